"""How often would partial reorthogonalisation (Simon's omega recurrence)
trigger on a config?  Runs the recurrence on the alpha/beta of a GPU build (full reorth).

  python tools/pro_estimate.py [--config 2] [--eps 6e-8]
"""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1803_06058_b200 import LoveCache
from synth import get_config, make_inputs


def simulate(alpha, beta, eps, thresh):
    k = len(alpha)
    w_prev = np.zeros(k + 1)       # omega_{j-1, .}
    w_cur = np.zeros(k + 1)        # omega_{j, .}
    w_cur[0] = 1.0
    trig, force = [], False
    for j in range(k - 1):
        b = beta[j]
        w_new = np.zeros(k + 1)
        for i in range(j):
            t = beta[i] * w_cur[i + 1] + (alpha[i] - alpha[j]) * w_cur[i] - (beta[j - 1] * w_prev[i] if j > 0 else 0.0)
            if i > 0:
                t += beta[i - 1] * w_cur[i - 1]
            w_new[i] = (t + np.sign(t) * eps * (beta[i] + b)) / b
        w_new[j] = eps
        w_new[j + 1] = 1.0
        if force or np.max(np.abs(w_new[:j + 1])) > thresh:
            trig.append(j)
            w_new[:j + 1] = eps
            w_cur[:j] = eps
            force = not force
        w_prev, w_cur = w_cur, w_new
    return trig


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--eps", type=float, default=6e-8)
    a = ap.parse_args()
    p = get_config(a.config)
    inp = make_inputs(p)
    c = LoveCache.build(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k,
                        precision=p.precision)
    info = c.info()
    for th in [np.sqrt(a.eps), 1e-5, 1e-6]:
        t = simulate(info["alpha"], info["beta"], a.eps, th)
        print(p.name, "threshold %.1e" % th, "reorth steps", len(t), "of", info["k_eff"] - 1, t[:40])


if __name__ == "__main__":
    main()
