"""One warm-up build + one profiled build and query of a config (for ncu launch lists).

  python tools/profile_build.py [--config 2] [--reps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1803_06058_b200 import LoveCache  # noqa: E402
from synth import get_config, make_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    p = get_config(a.config)
    inp = make_inputs(p)
    X = torch.from_numpy(inp.X).cuda()
    y = torch.from_numpy(inp.y).cuda()
    Xs = torch.from_numpy(inp.Xs).cuda()
    for _ in range(1 + a.reps):
        c = LoveCache.build(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k,
                            precision=p.precision)
        v = c.predict_var(Xs)
        torch.cuda.synchronize()
        c.free()
    print("ok", float(v.float().mean()))


if __name__ == "__main__":
    main()
