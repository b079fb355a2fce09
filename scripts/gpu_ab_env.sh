# A/B of runtime switches on one box: parity suite once, then bench garden (+ CONFIGS) per setting
#   TAG=t ENVS="MVGS_TMA=0|MVGS_TMA=1" CONFIGS="playroom" bash scripts/gpu_ab_env.sh
set -x
mkdir -p gpurun_out
T=${TAG:-ab}
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest.log
IFS='|' read -ra ES <<< "${ENVS}"
for r in 1 2; do
  i=0
  for e in "${ES[@]}"; do
    env $e timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_e${i}_r$r.json 2>&1
    for c in ${CONFIGS:-}; do env $e timeout 600 python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/${T}_e${i}_${c}_r$r.json 2>&1; done
    i=$((i+1))
  done
done
tail -2 gpurun_out/${T}_pytest.log
for f in gpurun_out/${T}_e*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); s=d['roofline']['stage_ms']
print('$f', d['value'], d['ms_per_step'], s['render_fwd'], s['render_bwd'])" 2>&1 | tail -1; done
