# A/B timing helper for gpurun: bench.py lines for a few env/library variants, interleaved
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])'
for rep in 1 2 3; do
 for v in ${ABVARS:-"fused:" "sep:LOVE_NO_FUSED_FFT=1"}; do
  n=${v%%:*}; e=${v#*:}; echo -n "$n $ABARGS " >> gpurun_out/${ABLOG:-ab.log}; env $e timeout 300 $B $ABARGS 2>/dev/null | python -c "$P" >> gpurun_out/${ABLOG:-ab.log}
 done
done
