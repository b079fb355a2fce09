# gpurun session: the NEXT-row benches (partial rendering Table-4 analog, D-SSIM, ADC step, variance lab)
set -x
mkdir -p gpurun_out
T=${TAG:-aux}
timeout 600 python bench_partial.py > gpurun_out/${T}_partial.log 2>&1
timeout 600 python bench_dssim.py > gpurun_out/${T}_dssim.log 2>&1
timeout 600 python bench_adc.py > gpurun_out/${T}_adc.log 2>&1
timeout 900 python bench_variance.py > gpurun_out/${T}_variance.log 2>&1
tail -1 gpurun_out/${T}_partial.log; tail -1 gpurun_out/${T}_dssim.log; tail -1 gpurun_out/${T}_adc.log; tail -1 gpurun_out/${T}_variance.log
