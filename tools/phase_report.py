"""Build / query timing per config and Lanczos mode, with the per-phase breakdown.

  python tools/phase_report.py [--configs 2,3,4,5] [--modes two_pass,one_read] [--reps 5]

Prints one JSON line per (config, mode): build ms (graph replay, CUDA events, median of
reps, L2 flushed before each), predict_var ms, and the eager per-phase ms of one build.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_06058_b200 import LoveCache, _abi  # noqa: E402
from synth import get_config, make_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--modes", default="two_pass,one_read")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    lib = _abi.load()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for ci in [int(x) for x in a.configs.split(",")]:
        p = get_config(ci)
        inp = make_inputs(p)
        X = torch.from_numpy(inp.X).cuda()
        y = torch.from_numpy(inp.y).cuda()
        Xs = torch.from_numpy(inp.Xs).cuda()
        for mode in a.modes.split(","):
            if mode == "one_read" and (p.precision != "fp32" or p.kind == "additive"):
                continue
            kw = dict(precision=p.precision)
            if p.kind != "additive":
                kw["lanczos_mode"] = mode
            try:
                c = (LoveCache.build_additive if p.kind == 'additive' else LoveCache.build)(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k, **kw)
                c.free()
            except Exception as e:  # report and continue
                print(json.dumps({"config": p.name, "mode": mode, "error": str(e)}), flush=True)
                continue
            bms, qms = [], []
            for _ in range(a.reps):
                flush.zero_()
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
                c = (LoveCache.build_additive if p.kind == 'additive' else LoveCache.build)(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k, **kw)
                e1.record()
                c.predict_var(Xs)
                e2.record()
                e2.synchronize()
                bms.append(e0.elapsed_time(e1))
                qms.append(e1.elapsed_time(e2))
                info = c.info()
                c.free()
            lib.love_profile_read(None, None, 1)
            lib.love_profile_enable(1)
            c = (LoveCache.build_additive if p.kind == 'additive' else LoveCache.build)(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k, **kw)
            c.predict_var(Xs)
            torch.cuda.synchronize()
            c.free()
            lib.love_profile_enable(0)
            ms = (ctypes.c_double * len(_abi.PROF_NAMES))()
            lib.love_profile_read(ms, None, 1)
            print(json.dumps({
                "config": p.name, "mode": mode, "k_eff": info["k_eff"],
                "build_ms_median": float(np.median(bms)), "build_ms_all": [round(b, 3) for b in bms],
                "query_ms_median": float(np.median(qms)), "t": p.t,
                "phase_ms_eager": {nm: round(ms[i], 4) for i, nm in enumerate(_abi.PROF_NAMES) if ms[i] > 0},
            }), flush=True)


if __name__ == "__main__":
    main()
