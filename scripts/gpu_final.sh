# gpurun session: per-config bench lines + ncu launch list of one garden step (for profiles/)
set -x
mkdir -p gpurun_out
T=${TAG:-fin}
for c in garden train playroom large; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_cfg_$c.json 2> gpurun_out/${T}_cfg_$c.err
done
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --profile --no-cpu-baseline --warmup 1 > gpurun_out/${T}_prof.log 2>&1
ls gpurun_out
