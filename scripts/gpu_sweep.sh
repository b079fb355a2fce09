# views-per-batch sweep at garden shape (Table 6 throughput analog, SURVEY §8(d) run matrix)
set -x
mkdir -p gpurun_out
T=${TAG:-sw}
for v in 1 2 4 8 16; do timeout 600 python bench.py --no-cpu-baseline --views $v --steps 10 > gpurun_out/${T}_views$v.log 2>&1; done
