"""Micro-benchmark of the K_UU MVM (love_kuu_mvm) and SKI MVM on a config's grid."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_06058_b200 import LoveCache  # noqa: E402
from synth import get_config, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
p = get_config(a.config)
inp = make_inputs(p)
c = LoveCache.build(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, 2, precision="fp64")
u = torch.randn(p.m_total, dtype=torch.float64, device="cuda")
v = torch.randn(p.n, dtype=torch.float64, device="cuda")
for name, fn, arg in [("kuu", c.kuu_mvm, u), ("ski", c.ski_mvm, v)]:
    for _ in range(10):
        fn(arg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn(arg)
    e1.record()
    e1.synchronize()
    print(f"{p.name} {name}_mvm: {e0.elapsed_time(e1) / a.iters * 1e3:.1f} us/call")
