# round-2 gpurun session: GPU tests, bench, optional per-config bench lines and ncu launch list
#   TAG=t1 TESTS=1 CONFIGS="train playroom" LAUNCHES=1 bash scripts/gpu_r2.sh
set -x
mkdir -p gpurun_out
T=${TAG:-t}
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest.log
fi
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for c in ${CONFIGS:-}; do timeout 600 python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/${T}_cfg_$c.json 2> gpurun_out/${T}_cfg_$c.err; done
if [ "${LAUNCHES:-0}" = 1 ]; then
  timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --profile --no-cpu-baseline --warmup 1 > gpurun_out/${T}_prof.log 2>&1
fi
if [ -n "${KREGEX:-}" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${KREGEX}" --launch-skip ${SKIP:-2} -c ${COUNT:-1} -o gpurun_out/${T}_full python bench.py --profile --no-cpu-baseline --warmup 1 --config ${CFG:-garden} > gpurun_out/${T}_full.log 2>&1
fi
tail -3 gpurun_out/${T}_pytest.log 2>/dev/null; python -c "
import json,sys
d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], json.dumps(d['roofline']['stage_ms']))" 2>&1 | tail -3
