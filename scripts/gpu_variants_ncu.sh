# A/B compile-time variants by ncu launch list (one profiled step each; kernel times, not a bench value)
#   TAG=v1 VARIANTS="|-DMVGS_SCAN_T=256" bash scripts/gpu_variants_ncu.sh
set -x
mkdir -p gpurun_out
T=${TAG:-varn}
IFS='|' read -ra VS <<< "${VARIANTS}"
i=0
for v in "${VS[@]}"; do
  MVGS_NVCC_EXTRA="$v" python -c "import sys; sys.path.insert(0,'paper_2506_12727_b200'); import build; build.build(force=True)" > gpurun_out/${T}_build$i.log 2>&1
  echo "variant[$i]: '$v'" > gpurun_out/${T}_v$i.log
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q >> gpurun_out/${T}_v$i.log 2>&1
  timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches$i.csv python bench.py --profile --no-cpu-baseline --warmup 1 >> gpurun_out/${T}_v$i.log 2>&1
  i=$((i+1))
done
python -c "import sys; sys.path.insert(0,'paper_2506_12727_b200'); import build; build.build(force=True)" > /dev/null 2>&1
