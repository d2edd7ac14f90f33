"""Config 5 breakdown-regime probe: k_eff, build time and variance error vs the fp64 oracle
for the fp32 build (several breakdown tolerances), the fp64 cache and the fp64 build."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_1803_06058_b200 import LoveCache  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402


def main():
    p = CONFIGS[5]
    inp = make_inputs(p)
    X, y, Xs = (torch.from_numpy(a).cuda() for a in (inp.X, inp.y, inp.Xs))
    model = O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)
    t0 = time.time()
    oc = O.love_precompute(model, p.k)
    print("oracle build s", round(time.time() - t0, 2), "k_eff", oc.lanczos.k_eff, flush=True)
    ov = O.predict_var(model, oc, inp.Xs)
    ia, wa = O.interp(inp.Xs, p.m, p.lo, p.h)
    prior = O.prior_ski(model, ia, wa, ia, wa)
    variants = [dict(precision="fp32", cache_fp64=False), dict(precision="fp32", cache_fp64=False, breakdown_tol=2e-7),
                dict(precision="fp32", cache_fp64=False, breakdown_tol=1e-7), dict(precision="fp32", cache_fp64=True),
                dict(precision="fp32"), dict(precision="fp64")]
    for kw in variants:
        for ks in (0, p.k_sample):
            def mk():
                return LoveCache.build(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k,
                                       k_sample=ks, **kw)
            c = mk()
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                c2 = mk()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
                c2.free()
            info = c.info()
            v = c.predict_var(Xs).double().cpu().numpy()
            rel = np.abs(v - ov) / np.abs(ov)
            b = np.abs(v - ov) / (1e-3 * np.abs(ov) + 1e-6 * prior)
            print(kw, "ks", ks, "k_eff", info["k_eff"], "ks_eff", info["k_sample_eff"],
                  "build ms %.3f" % np.median(ts), "maxrel %.3e" % rel.max(), "medrel %.3e" % np.median(rel),
                  "max/A21 %.3f" % b.max(), flush=True)
            c.free()


if __name__ == "__main__":
    main()
