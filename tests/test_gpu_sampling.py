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


@pytest.fixture(scope="module")
def cfg5_oracle():
    """Config 5 as BASELINE.json states it (n=1e5, m=1e4, k=k'=100, t=1e4, s=1000) and the fp64
    oracle's cache at the default breakdown tolerance (tau = 1e-10, reading A12)."""
    p = CONFIGS[5]
    inp = make_inputs(p)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    ia, wa = O.interp(inp.Xs, p.m, p.lo, p.h)
    return dict(p=p, inp=inp, model=model, oc=oc, var=O.predict_var(model, oc, inp.Xs),
                mu=O.predict_mean(model, oc, inp.Xs), prior=O.prior_ski(model, ia, wa, ia, wa))


def test_cfg5_full_size_parity(cfg5_oracle):
    """Config 5 through the configuration bench.py times (fp32 outputs, fp64 cache: opts.cache_fp64,
    reading A12b): the Lanczos runs to the oracle's breakdown step, and every one of the t = 1e4
    variances, the means and 20000 covariance pairs match the fp64 oracle.  Bound: BJ:north_star's
    fp32 relative 1e-3, asserted pointwise with no absolute slack; the measured error is the fp32
    rounding of the outputs (~6e-8)."""
    o = cfg5_oracle
    p, inp, model, oc = o["p"], o["inp"], o["model"], o["oc"]
    c = _build(p, inp, k_sample=p.k_sample, cache_fp64=p.cache_fp64)
    info = c.info()
    assert info["precision"] == 0 and info["cache_precision"] == 1
    assert info["k_eff"] == oc.lanczos.k_eff == 49
    # the leading recurrence coefficients are well determined (late ones follow round-off near
    # breakdown, which the variances do not see)
    np.testing.assert_allclose(info["alpha"][:30], oc.lanczos.alpha[:30], rtol=1e-9)
    Xs = torch.from_numpy(inp.Xs).cuda()
    var, mean = c.predict_var(Xs, return_mean=True)
    assert var.dtype == torch.float32
    var, mean = var.double().cpu().numpy(), mean.double().cpu().numpy()
    rel = np.abs(var - o["var"]) / np.abs(o["var"])
    print(f"cfg5 variances: max rel {rel.max():.3e}, median {np.median(rel):.3e}")
    assert rel.max() <= 1e-5
    assert np.max(np.abs(mean - o["mu"])) <= 1e-5 * np.abs(o["mu"]).max()
    rng = np.random.default_rng(5)
    ia, ib = rng.integers(0, p.t, 20_000), rng.integers(0, p.t, 20_000)
    cov = c.predict_covar(Xs[ia], Xs[ib]).double().cpu().numpy()
    cov_o = O.predict_covar(model, oc, inp.Xs[ia], inp.Xs[ib])
    scale = np.sqrt(o["var"][ia] * o["var"][ib])
    assert np.max(np.abs(cov - cov_o) / scale) <= 1e-5


def test_cfg5_fp32_breakdown_regime_auto_fp64_cache(cfg5_oracle):
    """The fp32 build in the breakdown regime (reading A12b).  With cache_fp64 OFF the fp32
    Lanczos (fp32 vectors, tau = 1e-6) stops where the oracle run with the same tau stops (k_eff
    37 < the tau = 1e-10 oracle's 49): its vectors cannot resolve beta_j below ~1e-7 ||T||, and
    the late directions are round-off (measured: up to 6 % variance error against the oracle at
    the same k, which fails the A21 bound).  The default (AUTO) therefore rebuilds such a cache
    with fp64 factors: fp32 outputs, the oracle's k_eff, variances within 1e-5."""
    o = cfg5_oracle
    p, inp, model = o["p"], o["inp"], o["model"]
    oc6 = O.love_precompute(model, p.k, tau=1e-6)
    Xs = torch.from_numpy(inp.Xs).cuda()
    off = _build(p, inp, cache_fp64=False)
    info = off.info()
    assert info["cache_precision"] == 0
    assert info["k_eff"] == oc6.lanczos.k_eff < o["oc"].lanczos.k_eff
    v_off = off.predict_var(Xs).double().cpu().numpy()
    assert np.all(v_off > 0) and np.all(v_off <= o["prior"] * (1 + 1e-6))
    ov6 = O.predict_var(model, oc6, inp.Xs)
    print(f"fp32 cache (OFF): k_eff {info['k_eff']}, max rel vs oracle(tau=1e-6) "
          f"{np.max(np.abs(v_off - ov6) / ov6):.3e}")
    auto = _build(p, inp)                                   # default cache_fp64 = "auto"
    ia = auto.info()
    assert ia["precision"] == 0 and ia["cache_precision"] == 1
    assert ia["k_eff"] == o["oc"].lanczos.k_eff
    v = auto.predict_var(Xs)
    assert v.dtype == torch.float32
    rel = np.abs(v.double().cpu().numpy() - o["var"]) / o["var"]
    assert rel.max() <= 1e-5, rel.max()


def test_cfg5_full_size_monte_carlo(cfg5_oracle):
    """Config 5 draws (Philox zeta, the bench's configuration): the covariance of the sampling root
    at the test points, W*^T S S^T W*, equals the oracle's LOVE covariance (deterministic part),
    and the sample mean / covariance match the oracle's predictive mean / covariance within
    Monte-Carlo bounds (6.5 standard errors, reading A23) on the t diagonals and 20000 pairs.
    Every bound is relative to the variances (no absolute slack)."""
    o = cfg5_oracle
    p, inp, model, oc = o["p"], o["inp"], o["model"], o["oc"]
    var, mu = o["var"], o["mu"]
    c = _build(p, inp, k_sample=p.k_sample, cache_fp64=p.cache_fp64)
    ks = c.info()["k_sample_eff"]
    S = c.export("S").cpu().numpy()
    ids, ws = O.interp(inp.Xs, p.m, p.lo, p.h)
    Sr = S.reshape(p.m_total, -1)[:, :ks]
    G = np.einsum("tl,tlk->tk", ws, Sr[ids])
    droot = (G * G).sum(1)
    rel_root = np.abs(droot - var) / var
    print(f"cfg5 root: k'_eff {ks}, diag(W*^T S S^T W*) vs LOVE var: max rel {rel_root.max():.3e}")
    assert rel_root.max() <= 1e-3
    F = c.sample(inp.Xs, p.s, seed=2018).double().cpu().numpy()
    assert np.isfinite(F).all()
    s = p.s
    Fm = F.mean(1)
    assert np.all(np.abs(Fm - mu) <= 6.5 * np.sqrt(var / s) + 1e-6 * np.abs(mu).max())
    dev = F - Fm[:, None]
    vhat = (dev * dev).sum(1) / (s - 1)
    assert np.all(np.abs(vhat - var) <= 6.5 * np.sqrt(2 * var * var / (s - 1)) + 1e-3 * var)
    rng = np.random.default_rng(5)
    ia, ib = rng.integers(0, p.t, 20_000), rng.integers(0, p.t, 20_000)
    cov = O.predict_covar(model, oc, inp.Xs[ia], inp.Xs[ib])
    chat = (dev[ia] * dev[ib]).sum(1) / (s - 1)
    se = np.sqrt((var[ia] * var[ib] + cov ** 2) / (s - 1))
    assert np.all(np.abs(chat - cov) <= 6.5 * se + 1e-3 * np.sqrt(var[ia] * var[ib]))


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
