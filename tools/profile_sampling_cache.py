"""Two cfg5 builds with the sampling cache (for ncu launch lists of the sampling Lanczos)."""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1803_06058_b200 import LoveCache
from synth import get_config, make_inputs
p = get_config(5); inp = make_inputs(p)
for _ in range(2):
    c = LoveCache.build(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k, precision=p.precision, k_sample=p.k_sample)
    torch.cuda.synchronize(); c.free()
