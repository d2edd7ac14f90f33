"""k-sweep accuracy study (synthetic analogue of PAPER.md Fig. 2,
P:728-745): how the LOVE variance error falls with the number of Lanczos steps k.

For each config, caches are built on the GPU for k in a ladder and the predictive variances of
a fixed seeded subset of the config's test points are compared with the largest-k cache of the
ladder (run to breakdown or k_max).  Reported per k: SMAE (mean |var_k - var_ref| / var(y),
P:683-684, reading A22), the median and max relative error, the median variance, and the
fraction of points whose variance did not increase from the previous k (LOVE variances are
non-increasing in k in exact arithmetic).

  python tools/k_sweep.py [--configs 1,2,3,4,5] [--ks 5,10,25,50,100,200,400] [--points 100000]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_06058_b200 import LoveCache  # noqa: E402
from synth import get_config, make_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--ks", default="5,10,25,50,100,200,400")
    ap.add_argument("--points", type=int, default=100_000)
    a = ap.parse_args()
    ks = [int(x) for x in a.ks.split(",")]
    for ci in [int(x) for x in a.configs.split(",")]:
        p = get_config(ci)
        inp = make_inputs(p)
        sel = np.random.default_rng(11).choice(p.t, min(a.points, p.t), replace=False)
        Xs = torch.from_numpy(inp.Xs[sel]).cuda()
        X = torch.from_numpy(inp.X).cuda()
        y = torch.from_numpy(inp.y).cuda()
        vy = float(np.var(inp.y))
        res = {}
        for k in ks:
            c = LoveCache.build(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, k,
                                precision=p.precision)
            v = c.predict_var(Xs).double().cpu().numpy()
            res[k] = (v, c.info()["k_eff"])
            c.free()
        kref = ks[-1]
        vref = res[kref][0]
        prev = None
        rows = []
        for k in ks:
            v, keff = res[k]
            err = np.abs(v - vref)
            row = {"config": p.name, "k": k, "k_eff": keff, "smae_vs_kref": float(err.mean() / vy),
                   "rel_err_median": float(np.median(err / np.abs(vref))),
                   "rel_err_max": float(np.max(err / np.abs(vref))), "var_median": float(np.median(v)),
                   "k_ref": kref, "k_ref_eff": res[kref][1], "points": int(len(sel))}
            if prev is not None:
                # non-increasing in k up to fp32 round-off of O(prior) terms
                row["frac_monotone"] = float(np.mean(v <= prev + 1e-5 * np.maximum(1.0, np.abs(prev))))
            prev = v
            rows.append(row)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
