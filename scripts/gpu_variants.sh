# A/B compile-time variants: bench garden with each MVGS_NVCC_EXTRA setting.  Each variant is
# built into its own library (MVGS_LIB), so the product libmvgs.so is never overwritten.
#   TAG=v1 CONFIGS="playroom" VARIANTS="|-DMVGS_RS_IPT=12|-DMVGS_RS_IPT=16" bash scripts/gpu_variants.sh
set -x
mkdir -p gpurun_out
T=${TAG:-var}
IFS='|' read -ra VS <<< "${VARIANTS}"
i=0
for v in "${VS[@]}"; do
  export MVGS_LIB=/tmp/mvgs_variant_$i.so
  MVGS_NVCC_EXTRA="$v" python -c "import sys; sys.path.insert(0,'paper_2506_12727_b200'); import build; build.build(force=True)" > gpurun_out/${T}_build$i.log 2>&1
  echo "variant[$i]: '$v'" > gpurun_out/${T}_v$i.log
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q >> gpurun_out/${T}_v$i.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline ${BENCH_ARGS} >> gpurun_out/${T}_v$i.log 2>&1
  for c in ${CONFIGS:-}; do timeout 600 python bench.py --no-cpu-baseline --config $c --steps 10 >> gpurun_out/${T}_v$i.log 2>&1; done
  unset MVGS_LIB
  i=$((i+1))
done
