# run one pytest selection under several compile-time variants
#   TAG=v3 VARIANTS="|-DMVGS_NO_CULL" SEL="tests/test_gpu_parity.py -k culling" bash scripts/gpu_variants_test.sh
set -x
mkdir -p gpurun_out
T=${TAG:-vt}
IFS='|' read -ra VS <<< "${VARIANTS}"
i=0
for v in "${VS[@]}"; do
  MVGS_NVCC_EXTRA="$v" python -c "import sys; sys.path.insert(0,'paper_2506_12727_b200'); import build; build.build(force=True)" > gpurun_out/${T}_build$i.log 2>&1
  echo "variant[$i]: '$v'" > gpurun_out/${T}_t$i.log
  timeout 600 python -m pytest ${SEL} -m gpu -q >> gpurun_out/${T}_t$i.log 2>&1
  i=$((i+1))
done
python -c "import sys; sys.path.insert(0,'paper_2506_12727_b200'); import build; build.build(force=True)" > /dev/null 2>&1
