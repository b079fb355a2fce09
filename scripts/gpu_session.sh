# one gpurun session: GPU tests, bench (default + every config), launch list
set -x
mkdir -p gpurun_out
T=${TAG:-s3}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
for c in train playroom large; do timeout 600 python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/${T}_bench_$c.log 2>&1; done
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --profile --no-cpu-baseline --warmup 1 > gpurun_out/${T}_prof.log 2>&1
tail -3 gpurun_out/${T}_pytest.log; tail -1 gpurun_out/${T}_bench.log
