# Round-end measurement set (profiles/): GPU suite, smoke, bench lines (garden + every config),
# ncu launch list of one step, ncu --set full of one whole step (per-stage DRAM traffic, and the
# compositing / per-Gaussian kernels' counters), the Table-4 analog and the scaling model.
set -x
mkdir -p gpurun_out
T=${TAG:-fin}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for c in train playroom large; do timeout 600 python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/${T}_cfg_$c.json 2> gpurun_out/${T}_cfg_$c.err; done
timeout 600 python bench.py --no-cpu-baseline --config large --scaling strong --exchange owner --steps 10 > gpurun_out/${T}_large_owner.json 2> gpurun_out/${T}_large_owner.err
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --profile --no-cpu-baseline --warmup 1 > gpurun_out/${T}_prof.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/${T}_step python bench.py --profile --no-cpu-baseline --warmup 1 > gpurun_out/${T}_step.log 2>&1
timeout 600 python bench_partial.py > gpurun_out/${T}_partial.json 2>&1
timeout 900 python bench_scaling.py > gpurun_out/${T}_scaling.json 2>&1
tail -2 gpurun_out/${T}_pytest.log; tail -1 gpurun_out/${T}_smoke.log
