"""cfg5: one warm sampling cache, then 3 draw calls (for ncu launch lists of the draw path)."""
import sys
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
from paper_1803_06058_b200 import LoveCache  # noqa: E402
from synth import get_config, make_inputs  # noqa: E402
p = get_config(5)
inp = make_inputs(p)
Xs = torch.from_numpy(inp.Xs).cuda()
c = LoveCache.build(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k,
                    precision=p.precision, k_sample=p.k_sample, cache_fp64=p.cache_fp64)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(3):
    c.sample(Xs, p.s, seed=0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
