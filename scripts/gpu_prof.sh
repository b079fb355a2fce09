# gpurun session: GPU tests, garden bench, ncu --set full of selected kernels on a config
#   TAG=s5 CFG=playroom KREGEX='k_render_bwd_w|k_render_fwd_p' bash scripts/gpu_prof.sh
set -x
mkdir -p gpurun_out
T=${TAG:-sx}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${KREGEX:-k_render_bwd_w}" --launch-skip ${SKIP:-2} -c ${COUNT:-2} -o gpurun_out/${T}_full python bench.py --profile --no-cpu-baseline --warmup 1 --config ${CFG:-garden} > gpurun_out/${T}_full.log 2>&1
tail -3 gpurun_out/${T}_pytest.log; tail -1 gpurun_out/${T}_bench.log
