# gpurun session: launch list + ncu --set full of every kernel of one garden step (for profiles/)
set -x
mkdir -p gpurun_out
T=${TAG:-fp}
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --profile --no-cpu-baseline --warmup 1 > gpurun_out/${T}_prof.log 2>&1
# the timed step's launches: skip the sizing pass + warm-up step (launch counts from the list)
timeout 1500 ncu --set full --import-source on --clock-control none --launch-skip ${SKIP:-62} -c ${COUNT:-22} -o gpurun_out/${T}_full python bench.py --profile --no-cpu-baseline --warmup 1 > gpurun_out/${T}_full.log 2>&1
tail -1 gpurun_out/${T}_bench.log
