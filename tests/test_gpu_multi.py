"""Multi-GPU: the training points of one problem sharded over 2 GPUs
(one process per GPU, liblove's NCCL all-reduces per Lanczos step) give the single-GPU cache
to fp32 round-off -- same k_eff, the same T, replicated caches on every rank, variances and
means within the A21 bound of the 1-GPU build and of the oracle.  Skipped below 2 GPUs (the
build's gpurun boxes have one; the gloo tests cover the host plumbing on CPU)."""
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import _gpu_multi_workers as W
import oracle as O
from synth import make_inputs, scaled_config

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs")]


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("ci,n,m,k,t", [(2, 60_001, (6000,), 40, 3001), (4, 60_013, (24, 24, 24), 40, 2005)])
def test_sharded_2gpu_equals_single_gpu(tmp_path, ci, n, m, k, t):
    from paper_1803_06058_b200 import LoveCache
    mp.spawn(W.sharded_equals_single, args=(2, _port(), ci, n, m, k, t, str(tmp_path)), nprocs=2, join=True)
    r = [np.load(tmp_path / f"rank{i}.npz") for i in range(2)]
    p = scaled_config(ci, n=n, m=m, k=k, t=t)
    g = make_inputs(p)
    c = LoveCache.build(g.X, g.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2, p.k)
    v1, m1 = (x.double().cpu().numpy() for x in c.predict_var(g.Xs, return_mean=True))
    i1 = c.info()
    for x in r:                                          # replicated caches
        assert int(x["k_eff"]) == i1["k_eff"] == k
        np.testing.assert_allclose(x["alpha"], i1["alpha"], rtol=1e-5)
    np.testing.assert_array_equal(r[0]["var"], r[1]["var"])
    model = O.build_model(g.X, g.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)
    ia, wa = O.interp(g.Xs, p.m, p.lo, p.h)
    prior = O.prior_ski(model, ia, wa, ia, wa)
    ov = O.predict_var(model, O.love_precompute(model, p.k), g.Xs)
    for ref in (v1, ov):
        err = np.abs(r[0]["var"] - ref)
        assert np.all(err <= 1e-3 * np.abs(ref) + 1e-6 * prior), np.max(err / (1e-3 * np.abs(ref) + 1e-6 * prior))
    assert np.max(np.abs(r[0]["mean"] - m1)) <= 1e-3 * np.abs(m1).max()
