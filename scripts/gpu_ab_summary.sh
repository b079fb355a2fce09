# Summary of a gpu_variants.sh run: parity result, garden and config step / render times per variant
#   TAG=w1 bash scripts/gpu_ab_summary.sh
T=${TAG:-var}
for f in gpurun_out/${T}_v*.log; do
  head -1 $f; grep -E "passed|failed" $f | tail -1
  python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{"metric"'):
        d = json.loads(l); s = d["roofline"]["stage_ms"]
        print(f'  {d["config"]["workload"][:10]:10s} {d["ms_per_step"]:.4f} ms  fwd {s["render_fwd"]:.4f} bwd {s["render_bwd"]:.4f} gauss {s["gauss_bwd"]:.4f}')
PY
done
