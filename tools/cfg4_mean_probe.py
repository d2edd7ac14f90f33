import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1803_06058_b200 import LoveCache
from synth import CONFIGS, make_inputs
p = CONFIGS[4]; inp = make_inputs(p)
d = np.load('/root/repo/tests/golden/cfg4_oracle_sample.npz')
X, y = (torch.from_numpy(a).cuda() for a in (inp.X, inp.y))
for mode in ("0", "1", "2"):
    os.environ["LOVE_AXIS_MMA"] = mode
    for cf in (False,):
        c = LoveCache.build(X, y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k, precision="fp32", cache_fp64=cf)
        v, mu = c.predict_var(torch.from_numpy(d["Xs"]).cuda(), return_mean=True)
        v = v.cpu().numpy().astype(np.float64); mu = mu.cpu().numpy().astype(np.float64)
        print("mode", mode, "k_eff", c.info()["k_eff"], "var maxrel %.3e" % np.max(np.abs(v - d["var"]) / np.abs(d["var"])),
              "mean err/max %.3e" % (np.max(np.abs(mu - d["mean"])) / np.abs(d["mean"]).max()), flush=True)
        c.free()
