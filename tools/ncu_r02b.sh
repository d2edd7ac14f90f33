# Round-2 evidence for the bench line: the launch list of the bench command (cold-cache,
# serialised: compare SHARES) and one ncu --set full capture of the dominant kernels (the
# reorthogonalisation dots + update of Lanczos step j = 49 of config 2, eager launches).
# Each command ran clean without ncu first (the && chains).
set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/r02_b2_plain.json && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_cfg2.csv $B > gpurun_out/r02_ncu_b2.log 2>&1
LOVE_NO_GRAPH=1 python tools/profile_build.py --config 2 && \
  LOVE_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:'reorth_(update|dots)' -s 98 -c 2 \
    -o gpurun_out/r02_reorth_cfg2 -f python tools/profile_build.py --config 2 > gpurun_out/r02_ncu_reorth.log 2>&1
