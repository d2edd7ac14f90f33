"""One-line summaries of bench.py JSON lines: python tools/bsum.py gpurun_out/b2.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e)
        continue
    s = d.get("sampling") or {}
    sr = (s.get("roofline") or {})
    print(f"{f}: {d['config']['workload']} ms/step {d['ms_per_step']:.3f} build {d['build_ms']:.3f} "
          f"query {d['query_ms']:.3f} k_eff {d.get('k_eff')} {d.get('cache_precision')} reorth {d['roofline']['frac']:.3f} "
          f"build {d['build_roofline']['frac']:.3f} query {d['query_roofline']['frac']:.3f} "
          f"value {d['value']:.3e} e2e {d['e2e']['value'] if d.get('e2e') else None}"
          + (f" sample {s['sample_ms']:.4f} ms frac {sr.get('frac')}" if s else ""))
    print("   ", d["phase_ms_per_step"])
