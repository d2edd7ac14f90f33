# A/B timing helper for gpurun: bench.py lines for a few env/library variants, interleaved
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])'
for rep in 1 2 3 4; do
 for v in "new:" "full:LOVE_FULL_EMBED=1" "base_full:LOVE_FULL_EMBED=1 LOVE_LIB=ab/liblove_base.so"; do
  n=${v%%:*}; e=${v#*:}; echo -n "$n " >> gpurun_out/ab_emb3.log; env $e timeout 300 $B $ABARGS 2>/dev/null | python -c "$P" >> gpurun_out/ab_emb3.log
 done
done
