"""In-pipeline per-kernel timing of the Lanczos step (graph replay + PDL, the production path):
runs tools/one_build.py under the trace build (liblove_trace.so, `make -C paper_1803_06058_b200
trace`) with LOVE_TRACE=1 and turns the library's trace line into a profile record.

Each kernel's slot = its first CTA start after griddepcontrol.wait -> the next kernel's first
start (%globaltimer), averaged over steps 2 .. k_eff - 3; the slots add up to the step period.
For the two reorthogonalisation passes the record adds the algorithmic bytes at the mean step
(dots (j+1) n v + n v, update (j+1) n v + 2 n v) and the fraction of the measured
HBM peak they reach inside the graph.

  python tools/trace_steps.py --configs 2 3 4 5 1 --out profiles/r02_trace
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import get_config  # noqa: E402


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
            if k in d:
                return float(d[k]), "measured (MEASURED_PEAKS.json %s)" % k
    except (OSError, ValueError):
        pass
    return 6544.3, "measured copy bandwidth recorded in round 1 (MEASURED_PEAKS.json absent)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_trace"))
    a = ap.parse_args()
    lib = os.path.join(ROOT, "paper_1803_06058_b200", "liblove_trace.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1803_06058_b200"), "-j", "8", "trace"], check=True)
    peak, peak_src = hbm_peak()
    for cfg in a.configs:
        env = dict(os.environ, LOVE_LIB=lib, LOVE_TRACE="1")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "one_build.py"), "--config", str(cfg)],
                           env=env, capture_output=True, text=True, check=True)
        lines = [ln for ln in r.stderr.splitlines() if ln.startswith('{"trace"')]
        # one_build.py builds twice (the second is the recorded one); a build prints the main
        # Lanczos line, then (k_sample > 0) the sampling Lanczos line
        per_build = 2 if getattr(get_config(cfg), "k_sample", 0) else 1
        lines = lines[-per_build:]
        tr = json.loads(lines[0])["trace"]
        p = get_config(cfg)
        rec = {"config": p.name, "n": p.n, "m": list(p.m), "k": p.k, "precision": p.precision,
               "source": "liblove_trace.so (LOVE_TRACE=1), tools/one_build.py --config %d, second build" % cfg,
               "steps": tr["steps"], "period_us": tr["period_us"], "slot_us": tr["slot_us"]}
        vs = 8 if (p.precision == "fp64" or getattr(p, "cache_fp64", False)) else 4
        steps = tr["steps"]
        if steps > 0 and "dots0" in tr["slot_us"] and "update0" in tr["slot_us"]:
            # steps 2 .. steps + 1 were averaged: mean j = (steps + 3) / 2
            jm = (steps + 3) / 2.0
            dots_b = (jm + 1) * p.n * vs + p.n * vs
            upd_b = (jm + 1) * p.n * vs + 2 * p.n * vs
            t = (tr["slot_us"]["dots0"] + tr["slot_us"]["update0"]) * 1e-6
            if vs == 8 and "dots1" in tr["slot_us"]:
                note = "fp64 CGS2: the DGKS-gated second pass is not counted in the bytes"
            else:
                note = "one CGS pass"
            rec["reorth_in_graph"] = {
                "mean_j": jm, "algorithmic_bytes_per_step": dots_b + upd_b,
                "slot_us": tr["slot_us"]["dots0"] + tr["slot_us"]["update0"],
                "achieved_gbs": (dots_b + upd_b) / t / 1e9, "peak_gbs": peak, "peak_source": peak_src,
                "frac": (dots_b + upd_b) / t / 1e9 / peak, "note": note}
        if per_build == 2:
            ts = json.loads(lines[1])["trace"]
            rec["sampling_lanczos"] = {"steps": ts["steps"], "period_us": ts["period_us"], "slot_us": ts["slot_us"],
                                       "note": "the M-Lanczos of the sampling cache (Eqs. 12-13); its step head is "
                                               "samp_qcur_dots (listed as 'moments')"}
        out = "%s_cfg%d.json" % (a.out, cfg)
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)
        print(json.dumps(rec))


if __name__ == "__main__":
    main()
