"""The buffers the build allocates without zero-fill (the Lanczos basis Q~ beyond its probe
column, the streamed cache columns Rc) are written before anything reads them:
with LOVE_POISON=1 the library fills them with NaN bytes at allocation instead, and the
cache must still match the fp64 oracle (a NaN read anywhere would propagate into the
variances).  Run in a subprocess because the library reads LOVE_POISON once per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, %(root)r)
import oracle as O
from paper_1803_06058_b200 import LoveCache
from synth import make_inputs, scaled_config

for ci, kw in ((1, dict(precision="fp64")), (2, dict(precision="fp32", n=20000, t=500, k=40)),
               (3, dict(precision="fp32", n=20000, t=500, k=40)), (4, dict(precision="fp32", n=5000, t=300, k=30)),
               (5, dict(precision="fp32", n=20000, t=500))):
    p = scaled_config(ci, **{k: v for k, v in kw.items() if k != "precision"}, precision=kw["precision"])
    inp = make_inputs(p)
    c = LoveCache.build(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k,
                        precision=p.precision)
    v = c.predict_var(inp.Xs).double().cpu().numpy()
    assert np.all(np.isfinite(v)), ci
    model = O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)
    oc = O.love_precompute(model, c.info()["k_eff"])
    ov = O.predict_var(model, oc, inp.Xs)
    ia, wa = O.interp(inp.Xs, model.m, model.lo, model.h)
    prior = O.prior_ski(model, ia, wa, ia, wa)
    a, b = (1e-9, 1e-13) if p.precision == "fp64" else (1e-3, 1e-6)
    err = np.abs(v - ov)
    assert np.all(err <= a * np.abs(ov) + b * prior), (ci, float(np.max(err / (a * np.abs(ov) + b * prior))))
    c.free()
print("POISON OK")
"""


def test_unset_buffers_are_written_before_read():
    env = dict(os.environ, LOVE_POISON="1")
    r = subprocess.run([sys.executable, "-c", _CHILD % {"root": ROOT}], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "POISON OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
