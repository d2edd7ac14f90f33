"""Parity of the CUDA path (through the C ABI) with the fp64 oracle, element by element on the
same seeded inputs.  Tolerances (reading A21):
  fp64 mode: |v - v_or| <= 1e-9 |v_or| + 1e-13 P(x*)
  fp32 mode: |v - v_or| <= 1e-3 |v_or| + 1e-6  P(x*)
where P(x*) is the prior variance.  Operators (K_UU, SKI MVM) are compared in relative 2-norm.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import CONFIGS, make_inputs, scaled_config, tiny_problem

pytestmark = pytest.mark.gpu


def _love():
    from paper_1803_06058_b200 import LoveCache, LoveError
    return LoveCache, LoveError


def _model(p, inp):
    return O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)


def _build(p, inp, **kw):
    LoveCache, _ = _love()
    kw.setdefault("precision", p.precision)
    return LoveCache.build(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2,
                           kw.pop("k", p.k), **kw)


def _prior(model, X):
    ia, wa = O.interp(X, model.m, model.lo, model.h)
    return O.prior_ski(model, ia, wa, ia, wa)


def _assert_var(got, want, prior, fp64):
    a, b = (1e-9, 1e-13) if fp64 else (1e-3, 1e-6)
    err = np.abs(got - want)
    bound = a * np.abs(want) + b * prior
    worst = np.argmax(err / bound)
    assert np.all(err <= bound), (f"max err/bound {np.max(err / bound):.3g} at {worst}: got {got[worst]} "
                                  f"want {want[worst]} prior {prior[worst]}; "
                                  f"max rel {np.max(err / np.abs(want)):.3g}")


def _rel2(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ------------------------------------------------------------------ K_UU MVM
@pytest.mark.parametrize("case", [
    ("cfg1", 1, None, "fp64"), ("cfg1_fp32", 1, None, "fp32"), ("cfg5m", 5, None, "fp32"),
    ("cfg2m", 2, None, "fp32"), ("cfg3m", 3, None, "fp32"), ("cfg4m", 4, None, "fp32"),
    ("1d_4096", 1, (4096,), "fp32"), ("1d_2049_fp64", 1, (2049,), "fp64"), ("3d_odd", 4, (9, 10, 11), "fp64"),
    ("1d_65537_fp64", 1, (65537,), "fp64"), ("1d_70001", 1, (70001,), "fp32"),   # real-input half-length FFT
    # shortened circulant embedding (reading A25b: N >= m + b, c_b < 1e-30 c_0): cfg2's grid at
    # N = 2^17 instead of 2^18, cfg5's at 2^14 instead of 2^15, m = 2200 on the one-CTA 4096 path
    ("cfg2m_fp64", 2, None, "fp64"), ("cfg5m_fp64", 5, None, "fp64"), ("1d_2200_fp64", 1, (2200,), "fp64"),
    # N = 2^18 and 2^19: the real-input half-length passes (rfft_passA/B/C, N >= 2^18)
    ("1d_200000", 2, (200_000,), "fp32"), ("1d_200000_fp64", 2, (200_000,), "fp64"),
    ("1d_300007_fp64", 2, (300_007,), "fp64"),
    # per-axis products on the FP64 tensor cores (L a multiple of 64): 32- and 16-column tiles,
    # several 64-row tiles, the last (contiguous) axis and a grid that mixes them with FFT axes
    ("cfg3m_fp64", 3, None, "fp64"), ("cfg4m_fp64", 4, None, "fp64"), ("3d_mma_fp64", 4, (128, 64, 192), "fp64"),
    ("2d_mixed_fp64", 3, (96, 64), "fp64"),
])
def test_kuu_mvm(case):
    name, ci, m, prec = case
    _kuu_mvm_case(ci, m, prec)


@pytest.mark.parametrize("mode", ["1", "2"])
def test_kuu_mvm_axis_products(mode, monkeypatch):
    """The dense per-axis products (DMMA / SIMT fp64) on every axis that tiles, at L = 64, 128,
    192, 256 (several 64-row tiles; LOVE_AXIS_MMA forces them where the FFT is the default),
    against the oracle's Toeplitz products in fp64."""
    monkeypatch.setenv("LOVE_AXIS_MMA", mode)
    _kuu_mvm_case(4, (128, 64, 192), "fp64")
    _kuu_mvm_case(3, None, "fp64")


def _kuu_mvm_case(ci, m, prec):
    p = scaled_config(ci, n=64, t=10, precision=prec, m=m, k=2)
    # training points only need to be valid: put them in the middle of the grid
    from synth.inputs import Inputs
    ctr = np.array([lo + (mm // 2 + 0.25) * h for lo, mm, h in zip(p.lo, p.m, p.h)])
    X = np.repeat(ctr[None, :], p.n, 0)
    y = np.random.default_rng(1).normal(size=p.n)
    c = _build(p, Inputs(X, y, X[:2]))
    rng = np.random.default_rng(7)
    u = rng.normal(size=p.m_total)
    got = c.kuu_mvm(torch.tensor(u, dtype=c.vdtype, device="cuda")).double().cpu().numpy()
    cols = [O.rbf_column(p.m[d], p.h[d], p.lengthscale[d]) for d in range(p.d)]
    want = O.kuu_matvec(cols, p.outputscale, u)
    tol = 1e-12 if prec == "fp64" else 2e-6 * max(1.0, np.log2(p.m_total))
    assert _rel2(got, want) < tol, _rel2(got, want)


# ------------------------------------------------------------------ SKI MVM
@pytest.mark.parametrize("case", [("1d_n40", "fp64"), ("1d_n200", "fp32"), ("2d", "fp64"), ("3d", "fp64"),
                                  ("2d", "fp32"), ("3d", "fp32")])
def test_ski_mvm_tiny(case):
    kind, prec = case
    p, inp = tiny_problem(kind)
    c = _build(p, inp, precision=prec, k=2)
    model = _model(p, inp)
    v = np.random.default_rng(3).normal(size=p.n)
    got = c.ski_mvm(torch.tensor(v, dtype=c.vdtype, device="cuda")).double().cpu().numpy()
    want = O.ski_mvm(model, v)
    assert _rel2(got, want) < (1e-12 if prec == "fp64" else 1e-5)


@pytest.mark.parametrize("ci,n,m", [(2, 50_003, (5000,)), (3, 40_001, (64, 64)), (4, 100_003, (24, 24, 24))])
def test_ski_mvm_scaled(ci, n, m):
    p = scaled_config(ci, n=n, m=m, k=2)
    inp = make_inputs(p)
    c = _build(p, inp)
    model = _model(p, inp)
    v = np.random.default_rng(5).normal(size=p.n)
    got = c.ski_mvm(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    want = O.ski_mvm(model, v)
    assert _rel2(got, want) < 1e-5


# ------------------------------------------------------------------ full LOVE pipeline
def test_cfg1_fp64_end_to_end():
    """Config 1 exactly as BASELINE.json states it (fp64, n=1000, m=256, k=50, t=1000)."""
    p = CONFIGS[1]
    inp = make_inputs(p)
    c = _build(p, inp)
    var, mean = c.predict_var(inp.Xs, return_mean=True)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    info = c.info()
    assert info["k_eff"] == oc.lanczos.k_eff
    k = info["k_eff"]
    np.testing.assert_allclose(info["alpha"], oc.lanczos.alpha[:k], rtol=1e-9)
    np.testing.assert_allclose(info["beta"][:k - 2], oc.lanczos.beta[:k - 2], rtol=1e-6)
    ov = O.predict_var(model, oc, inp.Xs)
    _assert_var(var.cpu().numpy(), ov, _prior(model, inp.Xs), fp64=True)
    om = O.predict_mean(model, oc, inp.Xs)
    np.testing.assert_allclose(mean.cpu().numpy(), om, atol=1e-9 * np.abs(om).max())
    # covariances of pairs (both priors): fp64 bound relative to sqrt(var_a var_b)
    Xb = inp.Xs[np.random.default_rng(2).permutation(p.t)]
    for prior in ("ski",):
        cov = c.predict_covar(inp.Xs, Xb).cpu().numpy()
        ocov = O.predict_covar(model, oc, inp.Xs, Xb, prior=prior)
        scale = np.sqrt(ov * O.predict_var(model, oc, Xb))
        _assert_cov(cov, ocov, scale, np.sqrt(_prior(model, inp.Xs) * _prior(model, Xb)), fp64=True)


def _assert_cov(got, want, scale, prior_scale, fp64):
    """Covariances: the A21 variance bound with |v_or| replaced by the covariance's own scale
    sqrt(var_a var_b) (>= |cov|) and P(x*) by sqrt(P_a P_b):
    fp64 1e-9 sqrt(v_a v_b) + 1e-13 sqrt(P_a P_b), fp32 1e-3 sqrt(v_a v_b) + 1e-6 sqrt(P_a P_b)."""
    a, b = (1e-9, 1e-13) if fp64 else (1e-3, 1e-6)
    r = np.abs(got - want) / (a * scale + b * prior_scale)
    assert r.max() <= 1.0, (r.max(), np.argmax(r))


@pytest.mark.parametrize("kind,prec", [("cfg1", "fp64"), ("cfg1", "fp32"), ("2d", "fp64"), ("3d", "fp64"),
                                       ("3d", "fp32")])
def test_prior_exact_covariances_distinct_points(kind, prec):
    """EXACT-prior mode (Eq. 10 with k(x*_i, x*_j), reading A8) on pairs of DISTINCT
    test points, product grids in 1-3-D, against the oracle's predict_covar(prior="exact") (its
    prior_exact is pinned to scikit-learn's RBF kernel in test_oracle_pins)."""
    if kind == "cfg1":
        # k = 30: config 1 converges (var << prior) and its fp32 Lanczos would stop before the
        # fp64 oracle's breakdown step (reading A12b)
        p = scaled_config(1, k=30, precision=prec)
        inp = make_inputs(p)
    else:
        import dataclasses as dc
        pt, inp = tiny_problem(kind)
        p = dc.replace(pt, k=60, precision=prec)
    c = _build(p, inp, prior="exact")
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    assert c.info()["k_eff"] == oc.lanczos.k_eff
    rng = np.random.default_rng(9)
    a, b = rng.integers(0, p.t, 3000), rng.integers(0, p.t, 3000)
    a, b = a[a != b], b[a != b]
    cov = c.predict_covar(inp.Xs[a], inp.Xs[b]).cpu().numpy().astype(np.float64)
    ocov = O.predict_covar(model, oc, inp.Xs[a], inp.Xs[b], prior="exact")
    va = O.predict_var(model, oc, inp.Xs[a], prior="exact")
    vb = O.predict_var(model, oc, inp.Xs[b], prior="exact")
    # EXACT-mode variances can be slightly negative where the SKI kernel's interpolation error
    # exceeds the variance (reading A8): the covariance scale uses |var|
    scale = np.sqrt(np.abs(va) * np.abs(vb))
    _assert_cov(cov, ocov, scale, np.full(len(a), p.outputscale), fp64=prec == "fp64")
    # the exact prior really is used: the result differs from the SKI-prior covariance by
    # k(x_a, x_b) - w_a^T K_UU w_b
    ia, wa = O.interp(inp.Xs[a], p.m, p.lo, p.h)
    ib, wb = O.interp(inp.Xs[b], p.m, p.lo, p.h)
    diff = O.prior_exact(model, inp.Xs[a], inp.Xs[b]) - O.prior_ski(model, ia, wa, ib, wb)
    cs = _build(p, inp).predict_covar(inp.Xs[a], inp.Xs[b]).cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(cov - cs, diff, atol=(1e-12 if prec == "fp64" else 1e-6) * p.outputscale)


@pytest.mark.parametrize("prec", ["fp64"])
def test_cfg1_probe_avgcol(prec):
    """Reading A1: the paper's own probe b = (1/m) W_X^T K_UU 1 (Alg. 1); the
    mean cache then follows Eq. 4, a = R^T T^{-1} Q^T y."""
    p = scaled_config(1, precision=prec)
    inp = make_inputs(p)
    c = _build(p, inp, probe="avg")
    var, mean = c.predict_var(inp.Xs, return_mean=True)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k, probe="avg")
    info = c.info()
    assert info["k_eff"] == oc.lanczos.k_eff
    np.testing.assert_allclose(info["b_norm"], oc.lanczos.b_norm, rtol=1e-12 if prec == "fp64" else 1e-6)
    ov = O.predict_var(model, oc, inp.Xs)
    _assert_var(var.cpu().numpy().astype(np.float64), ov, _prior(model, inp.Xs), fp64=prec == "fp64")
    om = O.predict_mean(model, oc, inp.Xs)
    tol = 1e-9 if prec == "fp64" else 1e-3
    assert np.max(np.abs(mean.cpu().numpy() - om)) <= tol * np.abs(om).max()


@pytest.mark.parametrize("mode", ["two_pass", "one_read"])
def test_scaled_cfg2_probe_avgcol(mode):
    p = scaled_config(2, n=60_001, m=(6000,), k=40, t=3001)
    inp = make_inputs(p)
    c = _build(p, inp, probe="avg", lanczos_mode=mode)
    var, mean = c.predict_var(inp.Xs, return_mean=True)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k, probe="avg")
    assert c.info()["k_eff"] == oc.lanczos.k_eff
    ov = O.predict_var(model, oc, inp.Xs)
    _assert_var(var.cpu().numpy().astype(np.float64), ov, _prior(model, inp.Xs), fp64=False)
    om = O.predict_mean(model, oc, inp.Xs)
    assert np.max(np.abs(mean.cpu().numpy() - om)) < 1e-3 * np.abs(om).max()


@pytest.mark.parametrize("mode", ["two_pass", "one_read"])
@pytest.mark.parametrize("ci,n,m,k,t", [
    (2, 60_001, (6000,), 40, 3001),          # 1-D four-step FFT, ragged n and t
    (3, 30_007, (48, 48), 40, 2003),         # 2-D Kronecker
    (3, 30_007, (64, 64), 40, 2003),         # 2-D, both axes on DMMA
    (4, 60_013, (24, 24, 24), 40, 2005),     # 3-D Kronecker
    (4, 60_013, (64, 32, 32), 40, 2005),     # 3-D, first axis on DMMA reading the scatter's sums (fuse_pull3)
    (5, 20_011, (2000,), 30, 1999),          # config-5 data, shorter grid
])
def test_scaled_fp32_variances_and_covariances(ci, n, m, k, t, mode):
    p = scaled_config(ci, n=n, m=m, k=k, t=t)
    inp = make_inputs(p)
    c = _build(p, inp, lanczos_mode=mode)
    var, mean = c.predict_var(inp.Xs, return_mean=True)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    info = c.info()
    assert info["k_eff"] == oc.lanczos.k_eff == k
    # fp32 Lanczos coefficients drift from the fp64 ones as j grows (finite-precision
    # Lanczos); the first steps must agree, the contract is on the variances.
    np.testing.assert_allclose(info["alpha"][:8], oc.lanczos.alpha[:8], rtol=1e-4)
    ov = O.predict_var(model, oc, inp.Xs)
    prior = _prior(model, inp.Xs)
    _assert_var(var.cpu().numpy().astype(np.float64), ov, prior, fp64=False)
    om = O.predict_mean(model, oc, inp.Xs)
    assert np.max(np.abs(mean.cpu().numpy() - om)) < 1e-3 * np.abs(om).max()
    # covariances on pairs (Xs[i], Xs[perm i])
    Xb = inp.Xs[np.random.default_rng(1).permutation(t)]
    cov = c.predict_covar(inp.Xs, Xb).cpu().numpy().astype(np.float64)
    ocov = O.predict_covar(model, oc, inp.Xs, Xb)
    scale = np.sqrt(prior * _prior(model, Xb))
    # fp32 caches form the pair products from fp64 rows of Rc, so the variance
    # bound's floor holds for covariances too: 1e-3 |cov| + 1e-6 sqrt(P_a P_b)
    ratio = np.abs(cov - ocov) / (1e-3 * np.abs(ocov) + 1e-6 * scale)
    assert ratio.max() <= 1.0, ratio.max()
    # symmetry cov(a,b) == cov(b,a)
    cov2 = c.predict_covar(Xb, inp.Xs).cpu().numpy().astype(np.float64)
    assert np.max(np.abs(cov - cov2)) <= 1e-6 * scale.max()


@pytest.mark.parametrize("kind", ["1d_n40", "1d_n200", "2d", "3d"])
def test_full_krylov_equals_dense_gp(kind):
    """fp64 GPU run to breakdown reproduces the dense-Cholesky SKI GP (north_star <= 1e-4 at k=n)."""
    p, inp = tiny_problem(kind)
    c = _build(p, inp, precision="fp64")
    var = c.predict_var(inp.Xs).cpu().numpy()
    model = _model(p, inp)
    _, dvar = O.dense_ski_gp(model, inp.Xs)
    assert c.info()["k_eff"] < p.k
    assert np.max(np.abs(var - dvar) / dvar) < 1e-6


# ------------------------------------------------------------------ edge cases
def test_edge_cases():
    LoveCache, LoveError = _love()
    p = scaled_config(1, n=301, t=5, k=10)
    inp = make_inputs(p)
    c = _build(p, inp)
    assert c.predict_var(np.zeros((0, 1))).numel() == 0                 # empty query batch
    bad = np.array([[-1.0], [0.5], [2.0]])                               # outside the grid
    v = c.predict_var(bad).cpu().numpy()
    assert np.isnan(v[0]) and np.isnan(v[2]) and np.isfinite(v[1])
    assert c.info()["n_out_of_range"] == 2
    with pytest.raises(LoveError) as e:                                   # training point off-grid
        LoveCache.build(np.array([[0.5], [1.2]]), np.ones(2), p.m, p.lo, p.h, p.lengthscale, 1.0, 0.01, 1)
    assert e.value.status == 2
    with pytest.raises(LoveError) as e:                                   # zero probe
        LoveCache.build(inp.X, np.zeros(p.n), p.m, p.lo, p.h, p.lengthscale, 1.0, 0.01, 3)
    assert e.value.status == 4
    c1 = _build(p, inp, k=1)                                              # k = 1
    assert c1.info()["k_eff"] == 1
    model = _model(p, inp)
    oc = O.love_precompute(model, 1)
    _assert_var(c1.predict_var(inp.Xs).cpu().numpy(), O.predict_var(model, oc, inp.Xs),
                _prior(model, inp.Xs), fp64=True)


def test_identity_like_breakdown():
    """All training points in one cell with equal weights -> the Krylov space of y under
    K_hat = W^T K W + s2 I has dimension <= 2: breakdown must stop at k_eff <= 2 (A12)."""
    p = scaled_config(1, n=64, t=4, k=10)
    X = np.full((64, 1), 0.5)
    y = np.random.default_rng(0).normal(size=64)
    LoveCache, _ = _love()
    c = LoveCache.build(X, y, p.m, p.lo, p.h, p.lengthscale, 1.0, 0.01, 10, precision="fp64")
    assert c.info()["k_eff"] <= 2
    from synth.inputs import Inputs
    model = _model(p, Inputs(X, y, X[:4]))
    oc = O.love_precompute(model, 10)
    assert oc.lanczos.k_eff == c.info()["k_eff"]
    _assert_var(c.predict_var(np.array([[0.3], [0.5]])).cpu().numpy(),
                O.predict_var(model, oc, np.array([[0.3], [0.5]])),
                _prior(model, np.array([[0.3], [0.5]])), fp64=True)


def test_prior_exact_mode():
    p = scaled_config(1, n=500, t=200, k=30)
    inp = make_inputs(p)
    c = _build(p, inp, prior="exact")
    var = c.predict_var(inp.Xs).cpu().numpy()
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    ov = O.predict_var(model, oc, inp.Xs, prior="exact")
    _assert_var(var, ov, np.full(len(ov), p.outputscale), fp64=True)


@pytest.mark.parametrize("one_sync", [True, False])
@pytest.mark.parametrize("ci,n,m,k", [(2, 50_003, (5000,), 30), (4, 40_009, (24, 24, 24), 25)])
def test_sharded_code_path_one_rank_nccl(ci, n, m, k, one_sync, monkeypatch):
    """The multi-GPU code path (every all-reduce issued through NCCL, eager step launches)
    with a one-rank communicator must give the single-GPU result: the collectives are
    identities, so any addressing or ordering bug in the sharded path shows up here.  fp32
    runs the one-sync step by default (one pass over Q~ for Q^T [r, q_j, q_{j-1}], three
    collectives per step); LOVE_NO_ONE_SYNC=1 the four-collective step.  Both
    also meet the oracle bound."""
    from paper_1803_06058_b200 import nccl_unique_id
    if not one_sync:
        monkeypatch.setenv("LOVE_NO_ONE_SYNC", "1")
    p = scaled_config(ci, n=n, m=m, k=k, t=2001)
    inp = make_inputs(p)
    c1 = _build(p, inp)
    cN = _build(p, inp, rank=0, world=1, nccl_id=nccl_unique_id())
    v1, m1 = c1.predict_var(inp.Xs, return_mean=True)
    vN, mN = cN.predict_var(inp.Xs, return_mean=True)
    assert cN.info()["k_eff"] == c1.info()["k_eff"]
    np.testing.assert_allclose(cN.info()["alpha"], c1.info()["alpha"], rtol=1e-6)
    np.testing.assert_allclose(vN.cpu().numpy(), v1.cpu().numpy(), rtol=1e-4, atol=1e-7)
    m1, mN = m1.cpu().numpy().astype(np.float64), mN.cpu().numpy().astype(np.float64)
    if one_sync:
        # a different (equally valid) fp32 CGS order: the mean, a Krylov solve (Eq. 3), moves
        # within the fp32 mean tolerance, measured ~5e-6 of max |mean|
        assert np.max(np.abs(mN - m1)) <= 1e-4 * np.abs(m1).max()
    else:
        np.testing.assert_allclose(mN, m1, rtol=1e-4, atol=1e-6)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    _assert_var(vN.cpu().numpy().astype(np.float64), O.predict_var(model, oc, inp.Xs), _prior(model, inp.Xs),
                fp64=False)
    om = O.predict_mean(model, oc, inp.Xs)
    assert np.max(np.abs(mN - om)) <= 1e-3 * np.abs(om).max()


@pytest.mark.parametrize("ci,n,m,k,prec", [(1, 1000, (256,), 50, "fp64"), (2, 60_001, (6000,), 40, "fp32"),
                                           (3, 30_007, (48, 48), 40, "fp32"), (5, 20_011, (2000,), 30, "fp32")])
@pytest.mark.parametrize("prior", ["ski", "exact"])
def test_var_blocks_vs_rc_rows_and_oracle(ci, n, m, k, prec, prior):
    """SURVEY 8(f) NEXT #3b: per-cell fp64 blocks B_c = (K_UU - Rc Rc^T)|stencil give the same
    Eq. 10 variances as the Rc-row path (reassociated), and both meet the oracle bound."""
    p = scaled_config(ci, n=n, m=m, k=k, t=4001, precision=prec)
    inp = make_inputs(p)
    cb = _build(p, inp, prior=prior)
    cr = _build(p, inp, prior=prior, var_blocks="off")
    vb, mb = cb.predict_var(inp.Xs, return_mean=True)
    vr, mr = cr.predict_var(inp.Xs, return_mean=True)
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    ov = O.predict_var(model, oc, inp.Xs, prior=prior)
    prior_v = _prior(model, inp.Xs)
    for v in (vb, vr):
        _assert_var(v.cpu().numpy().astype(np.float64), ov, prior_v, fp64=prec == "fp64")
    # means: same formula on both paths; the two builds differ only by fp64 atomic order
    np.testing.assert_allclose(mb.cpu().numpy(), mr.cpu().numpy(), rtol=1e-5, atol=1e-6)
    # the block path does the cancellation in fp64: in fp32 mode it is at least as close to
    # the oracle as the row path (median over points)
    eb = np.abs(vb.cpu().numpy().astype(np.float64) - ov)
    er = np.abs(vr.cpu().numpy().astype(np.float64) - ov)
    assert np.median(eb) <= np.median(er) * 1.5 + 1e-15


def test_sorted_queries_d3_match_unsorted_and_oracle(monkeypatch):
    """SURVEY 8(f) NEXT #3a: d = 3 variance queries counting-sorted by cell (64 Rc rows staged
    once per cell) equal the per-query path and the oracle; out-of-range points stay NaN."""
    p = scaled_config(4, n=60_013, m=(24, 24, 24), k=40, t=70_001)
    inp = make_inputs(p)
    Xs = inp.Xs.copy()
    Xs[17] = [9.0, 0.0, 0.0]                  # outside the grid -> NaN + counter
    Xs[40_000] = [0.0, -9.0, 0.0]
    c = _build(p, inp)
    vs, ms = c.predict_var(Xs, return_mean=True)
    monkeypatch.setenv("LOVE_NO_SORTED_QUERIES", "1")
    vu, mu = c.predict_var(Xs, return_mean=True)
    vs, ms, vu, mu = (x.cpu().numpy().astype(np.float64) for x in (vs, ms, vu, mu))
    bad = np.isnan(vu)
    assert bad.sum() == 2 and np.array_equal(np.isnan(vs), bad)
    np.testing.assert_allclose(vs[~bad], vu[~bad], rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(ms[~bad], mu[~bad], rtol=1e-5, atol=1e-7)
    assert c.info()["n_out_of_range"] == 4
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    sel = np.setdiff1d(np.arange(0, p.t, 13), [17, 40_000])
    ov = O.predict_var(model, oc, Xs[sel])
    _assert_var(vs[sel], ov, _prior(model, Xs[sel]), fp64=False)


def test_k_limit_is_an_argument_error():
    _, LoveError = _love()
    p, inp = tiny_problem("1d_n40")
    with pytest.raises(LoveError) as ei:
        _build(p, inp, k=4096)
    assert "k must be" in str(ei.value)


@pytest.mark.parametrize("ci,n,m,k,t", [(2, 60_001, (6000,), 40, 3001), (3, 30_007, (48, 48), 40, 2003)])
def test_partial_reorth_fp32_vs_full_oracle(ci, n, m, k, t):
    """partial reorthogonalisation (Simon's omega
    recurrence, one CGS pass when max|omega| > sqrt(eps_32)) keeps semi-orthogonality; far from
    convergence (the cfg2 / cfg3 regime at these k) its variances and means meet the same
    bounds against the fully reorthogonalised fp64 oracle.  Near convergence (cfg5's regime,
    var << prior) semi-orthogonality at sqrt(eps_32) is not enough for the 1e-3 bound, and the
    mode is documented as such."""
    p = scaled_config(ci, n=n, m=m, k=k, t=t)
    inp = make_inputs(p)
    c = _build(p, inp, lanczos_mode="partial")
    info = c.info()
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    assert info["k_eff"] == oc.lanczos.k_eff
    assert 0 <= info["n_reorth_steps"] < info["k_eff"] - 1
    var, mean = c.predict_var(inp.Xs, return_mean=True)
    ov = O.predict_var(model, oc, inp.Xs)
    _assert_var(var.cpu().numpy().astype(np.float64), ov, _prior(model, inp.Xs), fp64=False)
    om = O.predict_mean(model, oc, inp.Xs)
    assert np.max(np.abs(mean.cpu().numpy() - om)) < 1e-3 * np.abs(om).max()
    full = _build(p, inp)
    assert full.info()["n_reorth_steps"] == full.info()["k_eff"] - 1


def test_partial_reorth_is_fp32_single_gpu_only():
    _, LoveError = _love()
    p = CONFIGS[1]
    inp = make_inputs(p)
    with pytest.raises(LoveError):
        _build(p, inp, lanczos_mode="partial")          # fp64 config


@pytest.mark.parametrize("G", [2, 8])
def test_device_terminated_step_loop(monkeypatch, G):
    """The opt-in CUDA-graph WHILE loop (LOVE_COND_STEPS) stops on the device at breakdown:
    same k_eff, T and variances as the replayed step graph, and against the oracle.  Config-5
    shape (m = 10^4, k = 100) breaks down well before k."""
    from paper_1803_06058_b200 import launch_count
    p = scaled_config(5, n=30_011, k=100, t=2003, precision="fp64")
    inp = make_inputs(p)
    c0 = _build(p, inp)
    v0 = c0.predict_var(inp.Xs).cpu().numpy().astype(np.float64)
    i0 = c0.info()
    monkeypatch.setenv("LOVE_COND_STEPS", str(G))
    l0 = launch_count()
    c1 = _build(p, inp)
    l1 = launch_count() - l0
    v1 = c1.predict_var(inp.Xs).cpu().numpy().astype(np.float64)
    i1 = c1.info()
    assert i1["k_eff"] == i0["k_eff"] < p.k
    # fp64 atomics sum in a different order on every run: compare at the parity bounds
    np.testing.assert_allclose(i1["alpha"], i0["alpha"], rtol=1e-9)
    np.testing.assert_allclose(i1["beta"], i0["beta"], rtol=1e-6, atol=1e-9 * np.max(i0["beta"]))
    model = _model(p, inp)
    prior = _prior(model, inp.Xs)
    _assert_var(v1, v0, prior, fp64=True)
    # launches past the breakdown are not issued (at most G - 1 early-exiting steps run;
    # fp64: 9 kernels per step, two CGS passes)
    assert 0 < l1 < 9 * (i0["k_eff"] + G + 4) + 200
    oc = O.love_precompute(model, p.k)
    assert oc.lanczos.k_eff == i1["k_eff"]
    _assert_var(v1, O.predict_var(model, oc, inp.Xs), prior, fp64=True)


def test_sorted_queries_d3_large_k_falls_back(monkeypatch):
    """d = 3, t >= 65536 and a cache whose 64 stencil rows do not fit one CTA's shared memory
    (64 k_pad 8 B > 227 KB once k_pad > 443 in fp64): love_predict_var takes the per-query path
    instead of failing, and matches the oracle (query.cu smem cap)."""
    import dataclasses as dc
    p = dc.replace(scaled_config(4, n=6_007, m=(14, 14, 14), k=1024, t=70_001, precision="fp64"),
                   lo=(-4.5,) * 3, hi=(4.5,) * 3, lengthscale=(0.3, 0.3, 0.3))
    inp = make_inputs(p)
    c = _build(p, inp)
    k_eff = c.info()["k_eff"]
    assert k_eff > 443, k_eff
    v, mu = c.predict_var(inp.Xs, return_mean=True)
    monkeypatch.setenv("LOVE_NO_SORTED_QUERIES", "1")
    vu, muu = c.predict_var(inp.Xs, return_mean=True)
    np.testing.assert_array_equal(v.cpu().numpy(), vu.cpu().numpy())
    model = _model(p, inp)
    oc = O.love_precompute(model, p.k)
    # both run to breakdown; the step where beta_j crosses tau is set by round-off (+-3 steps
    # of directions that carry nothing)
    assert abs(oc.lanczos.k_eff - k_eff) <= 3
    sel = np.arange(0, p.t, 37)
    _assert_var(v.cpu().numpy()[sel], O.predict_var(model, oc, inp.Xs[sel]), _prior(model, inp.Xs[sel]), fp64=True)


def test_var_blocks2_pair_products_equal_warp_kernel(monkeypatch):
    """d = 2 variance blocks from node-pair products (query.cu pair_products2 + assembly) equal
    the warp-per-cell kernel's (LOVE_VAR_BLOCKS2_WARP=1): the same fp64 sums over the Rc
    columns, regrouped by node pair; both priors, with cells on the grid edge."""
    p = scaled_config(3, n=30_007, m=(48, 40), k=40, t=4001)
    inp = make_inputs(p)
    for prior in ("ski", "exact"):
        c = _build(p, inp, prior=prior)
        v = c.predict_var(inp.Xs).cpu().numpy().astype(np.float64)
        monkeypatch.setenv("LOVE_VAR_BLOCKS2_WARP", "1")
        cw = _build(p, inp, prior=prior)
        monkeypatch.delenv("LOVE_VAR_BLOCKS2_WARP")
        vw = cw.predict_var(inp.Xs).cpu().numpy().astype(np.float64)
        # the two builds differ only by fp64 atomic order in the Lanczos; the block algebra is
        # exact: fp32 outputs agree to round-off
        np.testing.assert_allclose(v, vw, rtol=2e-6, atol=1e-9)


@pytest.mark.parametrize("ci,n,m", [(1, 1000, (256,)), (3, 30_007, (48, 40))])
@pytest.mark.parametrize("prior", ["ski", "exact"])
def test_block_queries_cooperative_equal_per_thread(ci, n, m, prior, monkeypatch):
    """d <= 2 variance-block queries with G lanes per query (query.cu predict_block_coop_kernel,
    the default) equal the one-thread-per-query kernel (LOVE_QUERY_COOP=0) to fp64 summation
    order, means included, out-of-range points NaN in both (fp64 build)."""
    p = scaled_config(ci, n=n, m=m, k=30, t=5001, precision="fp64")
    inp = make_inputs(p)
    Xs = inp.Xs.copy()
    Xs[7] = 50.0                                       # outside the grid
    c = _build(p, inp, prior=prior)
    v, mu = (x.cpu().numpy() for x in c.predict_var(Xs, return_mean=True))
    monkeypatch.setenv("LOVE_QUERY_COOP", "0")                      # same cache, other kernel
    v2, mu2 = (x.cpu().numpy() for x in c.predict_var(Xs, return_mean=True))
    assert np.isnan(v[7]) and np.isnan(v2[7]) and np.isnan(mu[7])
    ok = ~np.isnan(v2)
    np.testing.assert_allclose(v[ok], v2[ok], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(mu[ok], mu2[ok], rtol=1e-10, atol=1e-14)


def test_cache_precision_options():
    """love_opts.cache_fp64 (reading A12b): ON gives an fp64 cache behind fp32 outputs (the
    operator and export dtypes follow the cache), OFF keeps fp32 even after a breakdown, ON
    with precision fp64 is an argument error; an fp32 problem that does not break down is not
    rebuilt under AUTO."""
    LoveCache, LoveError = _love()
    p = scaled_config(2, n=20_011, m=(2000,), k=20, t=501)
    inp = make_inputs(p)
    auto = _build(p, inp)
    assert auto.info()["k_eff"] == 20 and auto.info()["cache_precision"] == 0
    on = _build(p, inp, cache_fp64=True)
    i_on = on.info()
    assert i_on["precision"] == 0 and i_on["cache_precision"] == 1
    assert on.predict_var(inp.Xs).dtype == torch.float32
    assert on.export("rc").dtype == torch.float64
    v = np.random.default_rng(0).normal(size=p.n)
    mv = on.ski_mvm(torch.tensor(v, dtype=torch.float64, device="cuda"))
    assert mv.dtype == torch.float64
    np.testing.assert_allclose(mv.cpu().numpy(), O.ski_mvm(_model(p, inp), v), rtol=1e-11, atol=1e-11)
    with pytest.raises(LoveError) as e:
        _build(p, inp, precision="fp64", cache_fp64=True)
    assert e.value.status == 1
    # the fp64-cache variances equal the LOVE_FP64 build's, rounded to fp32
    f64 = _build(p, inp, precision="fp64")
    np.testing.assert_allclose(on.predict_var(inp.Xs).cpu().numpy(), f64.predict_var(inp.Xs).cpu().numpy(),
                               rtol=1e-6)
