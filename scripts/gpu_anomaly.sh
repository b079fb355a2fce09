# the MVGS_OS_IPT=16 render_bwd slowdown.  Builds the variant into its own
# library, benches it next to the default, captures render_bwd under ncu in both, and runs the
# parity tests of the variant under compute-sanitizer memcheck.  Also runs the ALU microbench.
set -x
mkdir -p gpurun_out
T=${TAG:-an}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_alu.cu && /tmp/mb > gpurun_out/${T}_alu.json 2>&1
/tmp/mb >> gpurun_out/${T}_alu.json 2>&1
export MVGS_LIB=/tmp/mvgs_ipt16.so
MVGS_NVCC_EXTRA="-DMVGS_OS_IPT=16" python -c "import sys; sys.path.insert(0,'paper_2506_12727_b200'); import build; build.build(force=True)" > gpurun_out/${T}_build.log 2>&1
for r in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_ipt16_bench$r.json 2>&1
  MVGS_LIB= timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_default_bench$r.json 2>&1
done
timeout 600 ncu --set full --clock-control none -k "regex:k_render_bwd|k_rs_onesweep" --launch-skip 0 -c 6 -o gpurun_out/${T}_ipt16 python bench.py --profile --no-cpu-baseline --warmup 1 --steps 1 > gpurun_out/${T}_ncu16.log 2>&1
MVGS_LIB= timeout 600 ncu --set full --clock-control none -k "regex:k_render_bwd|k_rs_onesweep" --launch-skip 0 -c 6 -o gpurun_out/${T}_ipt8 python bench.py --profile --no-cpu-baseline --warmup 1 --steps 1 > gpurun_out/${T}_ncu8.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not fullsize" > gpurun_out/${T}_memcheck16.log 2>&1
tail -3 gpurun_out/${T}_memcheck16.log
cat gpurun_out/${T}_alu.json
