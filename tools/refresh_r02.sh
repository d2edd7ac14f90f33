set -x
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
for c in 1 3 4 5 6; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rb$c.log 2> gpurun_out/rb$c.err; done
python tools/trace_steps.py --configs 2 3 4 5 1 --out gpurun_out/r02_trace > gpurun_out/trace_steps.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
