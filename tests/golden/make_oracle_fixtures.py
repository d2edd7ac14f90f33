"""Writes tests/golden/cfg4_oracle_sample.npz: the fp64 oracle's predictive variances for
config 4 at full size (n = 2e6, m = 64^3, k = 100) on 2000 seeded test points.

Calls only oracle/ and synth/ (no CUDA path).  Run from the repo root:
    python tests/golden/make_oracle_fixtures.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402


def main():
    p = CONFIGS[4]
    inp = make_inputs(p)
    model = O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)
    cache = O.love_precompute(model, p.k)
    sel = np.sort(np.random.default_rng(2024).choice(p.t, 2000, replace=False))
    Xs = inp.Xs[sel]
    var = O.predict_var(model, cache, Xs)
    mean = O.predict_mean(model, cache, Xs)
    ia, wa = O.interp(Xs, p.m, p.lo, p.h)
    prior = O.prior_ski(model, ia, wa, ia, wa)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg4_oracle_sample.npz")
    np.savez_compressed(out, Xs=Xs, var=var, mean=mean, prior=prior, alpha=cache.lanczos.alpha,
                        beta=cache.lanczos.beta, k_eff=cache.lanczos.k_eff)
    print("wrote", out, "k_eff", cache.lanczos.k_eff, "var median", np.median(var))


if __name__ == "__main__":
    main()
