"""Posterior sampling (Eqs. 11-15) against the oracle.

* deterministic part: the covariance implied by the sampling root, W*^T S S^T W*, equals the
  oracle's (fp64 build) at test points;
* shared draws: with the same zeta the samples equal the oracle's (fp64 build);
* Monte-Carlo part: Philox draws have the predictive mean and covariance within 6.5 standard
  errors, SE_ij = sqrt((C_ii C_jj + C_ij^2)/(s-1)) (SURVEY §8(c) sampling pin), and are
  deterministic per seed.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import CONFIGS, make_inputs, make_zeta, scaled_config, tiny_problem

pytestmark = pytest.mark.gpu


def _build(p, inp, **kw):
    from paper_1803_06058_b200 import LoveCache
    kw.setdefault("precision", p.precision)
    return LoveCache.build(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2,
                           kw.pop("k", p.k), **kw)


def _model(p, inp):
    return O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)


def _root_cov(p, S, ks_pad, ks, Xs):
    """W*^T S S^T W* from an exported row-major S (m x ks_pad)."""
    S = S.reshape(-1, ks_pad)[:, :ks].astype(np.float64)
    ids, ws = O.interp(Xs, p.m, p.lo, p.h)
    G = np.einsum("tl,tlk->tk", ws, S[ids])
    return G @ G.T


@pytest.mark.parametrize("kind,ks", [("1d_n200", 60), ("2d", 80)])
def test_sampling_root_covariance_vs_oracle(kind, ks):
    p, inp = tiny_problem(kind)
    c = _build(p, inp, precision="fp64", k_sample=ks)
    info = c.info()
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    sc = O.sampling_cache(model, oc, ks)
    # run past the numerical rank of M: both stop at breakdown (reading A12), which falls in
    # the tail of M's spectrum (52 eigenvalues above 1e-8 max|M|, 63 above 1e-12),
    # so k'_eff is set by round-off and may differ by a few steps; the extra directions carry
    # ~0 eigenvalues of T' and the contract is on S S^T below (reading A15)
    assert abs(info["k_sample_eff"] - sc.lanczos.k_eff) <= 5
    Xs = inp.Xs[:20]
    S = c.export("S").cpu().numpy()
    Cg = _root_cov(p, S, S.size // p.m_total, info["k_sample_eff"], Xs)
    ids, ws = O.interp(Xs, p.m, p.lo, p.h)
    Go = np.einsum("tl,tlk->tk", ws, sc.S[ids])
    Co = Go @ Go.T
    assert np.abs(Cg - Co).max() <= 1e-8 * np.abs(Co).max()


def test_shared_zeta_samples_match_oracle():
    # S = Q' T'^{1/2} itself (not only S S^T) must agree, so use the well-determined leading
    # Lanczos directions of M (late Lanczos vectors are sensitive to round-off)
    p = scaled_config(5, n=20_011, m=(2000,), k=40, t=300, k_sample=12, s=64)
    inp = make_inputs(p)
    c = _build(p, inp, precision="fp64", k_sample=p.k_sample)
    info = c.info()
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    sc = O.sampling_cache(model, oc, p.k_sample)
    assert info["k_sample_eff"] == sc.lanczos.k_eff == p.k_sample
    zeta = make_zeta(p.k_sample, p.s)
    F = c.sample(inp.Xs, p.s, zeta=zeta).cpu().numpy()
    Fo = O.draw_samples(model, oc, sc, inp.Xs, zeta)
    mu = O.predict_mean(model, oc, inp.Xs)
    dev = Fo - mu[:, None]
    # the sample GEMM runs in fp32 (FMA): round-off ~ 1e-6 of the deviations
    assert np.abs(F - Fo).max() <= 1e-5 * np.abs(dev).max() + 1e-6 * np.abs(mu).max()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_philox_samples_monte_carlo_and_determinism(precision):
    """The draws of the sampler have the mean and the covariance W*^T S S^T W* of the cache
    they were drawn from (Eq. 11), within Monte-Carlo bounds; fp64 builds' caches also equal
    the oracle's (test above), fp32 builds' caches inherit the fp32 LOVE cache's round-off."""
    p = scaled_config(5, n=20_011, m=(2000,), k=40, t=12, k_sample=40, s=40_000)
    inp = make_inputs(p)
    c = _build(p, inp, k_sample=p.k_sample, precision=precision)
    F1 = c.sample(inp.Xs, p.s, seed=7).double().cpu().numpy()
    F2 = c.sample(inp.Xs, p.s, seed=7).double().cpu().numpy()
    F3 = c.sample(inp.Xs, 64, seed=8).double().cpu().numpy()
    assert np.array_equal(F1, F2)
    assert not np.allclose(F1[:, :64], F3)
    S = c.export("S").cpu().numpy()
    C = _root_cov(p, S, S.size // p.m_total, c.info()["k_sample_eff"], inp.Xs)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    mu = O.predict_mean(model, oc, inp.Xs)
    s = p.s
    Chat = np.cov(F1)
    se = np.sqrt((np.outer(np.diag(C), np.diag(C)) + C ** 2) / (s - 1))
    assert np.all(np.abs(Chat - C) <= 6.5 * se + 1e-4 * np.abs(C).max())
    assert np.all(np.abs(F1.mean(1) - mu) <= 6.5 * np.sqrt(np.diag(C) / s) + 1e-4 * np.abs(mu).max())


def test_cfg5_full_size_monte_carlo():
    """Config 5 as BASELINE.json states it: n=1e5, m=1e4, k=k'=100, s=1000 joint samples at
    t=1e4 test points; sample mean / covariance vs the oracle's predictive mean / covariance
    (LOVE covariance, Eq. 10) within Monte-Carlo bounds on the t diagonals and 20000 pairs."""
    p = CONFIGS[5]
    inp = make_inputs(p)
    c = _build(p, inp, k_sample=p.k_sample)
    F = c.sample(inp.Xs, p.s, seed=2018).double().cpu().numpy()
    assert np.isfinite(F).all()
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    mu = O.predict_mean(model, oc, inp.Xs)
    var = O.predict_var(model, oc, inp.Xs)
    s = p.s
    Fm = F.mean(1)
    assert np.all(np.abs(Fm - mu) <= 6.5 * np.sqrt(var / s) + 1e-4 * np.abs(mu).max())
    dev = F - Fm[:, None]
    vhat = (dev * dev).sum(1) / (s - 1)
    assert np.all(np.abs(vhat - var) <= 6.5 * np.sqrt(2 * var * var / (s - 1)) + 1e-6)
    rng = np.random.default_rng(5)
    ia, ib = rng.integers(0, p.t, 20_000), rng.integers(0, p.t, 20_000)
    cov = O.predict_covar(model, oc, inp.Xs[ia], inp.Xs[ib])
    chat = (dev[ia] * dev[ib]).sum(1) / (s - 1)
    se = np.sqrt((var[ia] * var[ib] + cov ** 2) / (s - 1))
    assert np.all(np.abs(chat - cov) <= 6.5 * se + 1e-6)


def test_tridiag_root_matches_jacobi_root(monkeypatch):
    """The sampling root's eigensolver (multisection + twisted factorisation + CGS2 in
    clusters) against the cyclic Jacobi kernel (LOVE_JACOBI=1) on the same fp64 build, past
    breakdown so T' carries its cluster of ~0 eigenvalues: S S^T agrees to 1e-9 of its max."""
    p, inp = tiny_problem("1d_n200")
    S = {}
    for jac in (False, True):
        if jac:
            monkeypatch.setenv("LOVE_JACOBI", "1")
        c = _build(p, inp, precision="fp64", k_sample=60)
        ke = c.info()["k_sample_eff"]
        Sx = c.export("S").cpu().numpy().reshape(p.m_total, -1)[:, :ke]
        S[jac] = Sx @ Sx.T
    assert np.abs(S[False] - S[True]).max() <= 1e-9 * np.abs(S[True]).max()
