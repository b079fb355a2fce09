# A/B session: GPU tests, partial tests repeated, bench with and without evaluation counting
set -x
mkdir -p gpurun_out
T=${TAG:-ab}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest.log
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_partial.py -m gpu -q >> gpurun_out/${T}_partial.log 2>&1; done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
MVGS_BENCH_COUNT=1 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_count.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench2.log 2>&1
tail -3 gpurun_out/${T}_pytest.log; grep passed gpurun_out/${T}_partial.log
