# Round-2 ncu --set full captures of the kernels VERDICT r01 asked for (run under gpurun, one GPU).
# Every command ran clean without ncu first (the && chain).  Eager launches (LOVE_NO_GRAPH=1)
# so ncu sees every step kernel; --profile-from-start off: the second (warm) build of
# tools/one_build.py is profiled.  Step j = 49: skip 49 launches of each matched kernel group.
set -x
N="ncu --set full --clock-control none --import-source on --profile-from-start off"
export LOVE_NO_GRAPH=1
python tools/one_build.py --config 4 && \
  $N -k regex:'moments_kernel|gather_kernel|pull_last|pull_mid|pull_first' -s 245 -c 5 -o gpurun_out/r02_ski_cfg4 -f python tools/one_build.py --config 4 > gpurun_out/ncu4.log 2>&1
python tools/one_build.py --config 3 && \
  $N -k regex:'moments2_tpc|pull_last|pull_first|axis_conv|gather_pts1' -s 294 -c 6 -o gpurun_out/r02_ski_cfg3 -f python tools/one_build.py --config 3 > gpurun_out/ncu3.log 2>&1 && \
  $N -k regex:'pair_products|assemble_blocks|predict_block' -c 3 -o gpurun_out/r02_finish_query_cfg3 -f python tools/one_build.py --config 3 > gpurun_out/ncu3b.log 2>&1
python tools/one_build.py --config 2 && \
  $N -k regex:'predict_block|moments_cell1|gather_pts1' -s 98 -c 3 -o gpurun_out/r02_query_cfg2 -f python tools/one_build.py --config 2 > gpurun_out/ncu2.log 2>&1
python tools/one_build.py --config 4 && \
  $N -k regex:'predict_sorted3|query_cell3' -c 2 -o gpurun_out/r02_query_cfg4 -f python tools/one_build.py --config 4 > gpurun_out/ncu4q.log 2>&1
python tools/profile_draws.py && \
  $N -k regex:'sample_gemm2|sample_gather|philox' -c 3 -o gpurun_out/r02_draws_cfg5 -f python tools/profile_draws.py > gpurun_out/ncu5.log 2>&1
