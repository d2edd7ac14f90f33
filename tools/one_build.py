"""One warm build (+ predict_var) of a config inside cudaProfilerStart/Stop, for ncu launch lists:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --cache-control none --csv python tools/one_build.py --config 2

A first build runs outside the profiled range, so the profiled one sees warm caches and
already-instantiated graphs.
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
    ap.add_argument("--lanczos_mode", default="auto")
    a = ap.parse_args()
    p = get_config(a.config)
    inp = make_inputs(p)
    X = torch.from_numpy(inp.X).cuda()
    y = torch.from_numpy(inp.y).cuda()
    Xs = torch.from_numpy(inp.Xs).cuda()
    kw = dict(precision=p.precision)
    if p.kind == "additive":
        fn = LoveCache.build_additive
    else:
        fn = LoveCache.build
        kw["lanczos_mode"] = a.lanczos_mode
    if p.k_sample:
        kw["k_sample"] = p.k_sample
    if p.cache_fp64:
        kw["cache_fp64"] = True
    for it in range(2):
        if it == 1:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        c = fn(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k, **kw)
        c.predict_var(Xs)
        torch.cuda.synchronize()
        c.free()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
