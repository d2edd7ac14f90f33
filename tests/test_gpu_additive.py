"""Additive kernel compositions (Eq. 16) on the GPU, through
love_build_cache_additive, against the fp64 oracle (same tolerances as test_gpu_parity)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import make_inputs, scaled_config, tiny_problem

pytestmark = pytest.mark.gpu

S2 = [0.7, 1.3, 1.0]


def _love():
    from paper_1803_06058_b200 import LoveCache, LoveError
    return LoveCache, LoveError


def _s2(p):
    return S2[:p.d] if p.d <= 3 else [1.0] * p.d


def _model(p, inp):
    return O.build_model_additive(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, _s2(p), p.sigma2)


def _build(p, inp, **kw):
    LoveCache, _ = _love()
    kw.setdefault("precision", p.precision)
    return LoveCache.build_additive(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, _s2(p), p.sigma2,
                                    kw.pop("k", p.k), **kw)


def _prior(model, X):
    ia, wa = O.model_interp(model, X)
    return O.prior_ski(model, ia, wa, ia, wa)


def _assert_var(got, want, prior, fp64):
    a, b = (1e-9, 1e-13) if fp64 else (1e-3, 1e-6)
    err = np.abs(got - want)
    bound = a * np.abs(want) + b * prior
    assert np.all(err <= bound), (np.max(err / bound), np.max(err / np.abs(want)))


def test_additive_operators_fp64():
    p, inp = tiny_problem("additive3")
    model = _model(p, inp)
    c = _build(p, inp, k=3)
    u = np.random.default_rng(1).normal(size=model.m_total)
    got = c.kuu_mvm(torch.tensor(u, dtype=torch.float64, device="cuda")).cpu().numpy()
    want = O.model_kuu_matvec(model, u)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    v = np.random.default_rng(2).normal(size=p.n)
    got = c.ski_mvm(torch.tensor(v, dtype=torch.float64, device="cuda")).cpu().numpy()
    want = O.ski_mvm(model, v)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("prior", ["ski", "exact"])
def test_additive_full_krylov_equals_dense_gp(prior):
    """Run to breakdown, LOVE on the block forms equals the dense GP of the additive SKI
    kernel (Eq. 7 bridge) -- on the GPU through the C ABI."""
    p, inp = tiny_problem("additive3")
    model = _model(p, inp)
    c = _build(p, inp, prior=prior)
    oc = O.love_precompute(model, p.k)
    assert c.info()["k_eff"] == oc.lanczos.k_eff
    var, mean = c.predict_var(inp.Xs, return_mean=True)
    ov = O.predict_var(model, oc, inp.Xs, prior=prior)
    _assert_var(var.cpu().numpy(), ov, _prior(model, inp.Xs), fp64=True)
    md, vd = O.dense_ski_gp(model, inp.Xs)
    if prior == "ski":
        np.testing.assert_allclose(var.cpu().numpy(), vd, rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(mean.cpu().numpy(), md, rtol=1e-8, atol=1e-10)
    Xb = inp.Xs[::-1].copy()
    cov = c.predict_covar(inp.Xs, Xb).cpu().numpy()
    ocov = O.predict_covar(model, oc, inp.Xs, Xb, prior=prior)
    np.testing.assert_allclose(cov, ocov, rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("probe", ["y", "avg"])
def test_additive_cfg6_scaled_fp32(probe):
    """Config 6 shape (10 components, m = 100 each, Styblinski-Tang data) at n = 20,000."""
    p = scaled_config(6, n=20_011, k=40, t=3001)
    inp = make_inputs(p)
    model = _model(p, inp)
    c = _build(p, inp, probe=probe)
    oc = O.love_precompute(model, p.k, probe=probe)
    assert c.info()["k_eff"] == oc.lanczos.k_eff
    var, mean = c.predict_var(inp.Xs, return_mean=True)
    ov = O.predict_var(model, oc, inp.Xs)
    _assert_var(var.cpu().numpy().astype(np.float64), ov, _prior(model, inp.Xs), fp64=False)
    # covariances of an fp32 cache come from its fp64 row copy (Rc64): the variance bound with
    # sqrt(var_a var_b) and sqrt(P_a P_b) in place of |v| and P
    Xb = inp.Xs[::-1].copy()
    cov = c.predict_covar(inp.Xs, Xb).cpu().numpy().astype(np.float64)
    ocov = O.predict_covar(model, oc, inp.Xs, Xb)
    scale = np.sqrt(ov * O.predict_var(model, oc, Xb))
    pscale = np.sqrt(_prior(model, inp.Xs) * _prior(model, Xb))
    assert np.all(np.abs(cov - ocov) <= 1e-3 * scale + 1e-6 * pscale)
    om = O.predict_mean(model, oc, inp.Xs)
    assert np.max(np.abs(mean.cpu().numpy() - om)) < 1e-3 * np.abs(om).max()


def test_additive_edge_cases():
    LoveCache, LoveError = _love()
    p, inp = tiny_problem("additive3")
    c = _build(p, inp, k=20)
    Xs = inp.Xs[:5].copy()
    Xs[2, 1] = 50.0                                  # outside component 1's grid
    v = c.predict_var(Xs).cpu().numpy()
    assert np.isnan(v[2]) and np.all(np.isfinite(np.delete(v, 2)))
    assert c.info()["n_out_of_range"] == 1
    X = inp.X.copy()
    X[0, 2] = -50.0
    with pytest.raises(LoveError) as ei:
        LoveCache.build_additive(X, inp.y, p.m, p.lo, p.h, p.lengthscale, _s2(p), p.sigma2, 5, precision="fp64")
    assert "ERR_RANGE" in str(ei.value)
    from paper_1803_06058_b200 import _abi
    import ctypes
    axes = (_abi.love_axis * 3)()
    for e in range(3):
        axes[e].m, axes[e].lo, axes[e].h, axes[e].lengthscale, axes[e].outputscale = 15, -7.0, 1.0, 1.0, 1.0
    o = _abi.love_opts()
    o.k_sample = 5
    out = ctypes.c_void_p()
    Xd = torch.from_numpy(inp.X).cuda()
    yd = torch.from_numpy(inp.y).cuda()
    st = _abi.load().love_build_cache_additive(axes, 3, 0.01, ctypes.c_void_p(Xd.data_ptr()),
                                               ctypes.c_void_p(yd.data_ptr()), p.n, 5, ctypes.byref(o), None,
                                               None, ctypes.byref(out))
    assert st == _abi.LOVE_ERR_ARG and not out.value
