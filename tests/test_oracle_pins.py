"""Pins of the fp64 oracle to things other than itself (CPU only, `-m "not gpu"`).

Each test checks the oracle against a closed form, a hand-derived example
(tests/golden/spec_examples.json, with citations), a library routine that the oracle does
not use for that step, a mathematical invariant, or the dense-Cholesky GP.  A plausible
mistake (dropped term, wrong sign/index, transposed operand) fails at least one of them.
"""
import json
import math
import os
import types

import numpy as np
import pytest

import oracle as O
from synth import CONFIGS, make_inputs, scaled_config, tiny_problem

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _model(p, inp):
    return O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, p.sigma2)


# ---------------------------------------------------------------- interpolation
def test_keys_golden():
    for ex in GOLDEN["keys_weights"]:
        np.testing.assert_allclose(O.keys_weights(np.array([ex["f"]]))[0], ex["w"], atol=1e-15)


def test_keys_reproduces_quadratics():
    """Keys a=-1/2 interpolates 1, x and x^2 exactly (reading A2; X0): a wrong sign, a
    wrong `a` or a mis-ordered stencil breaks one of these moments."""
    f = np.random.default_rng(3).uniform(0, 1, 1000)
    w = O.keys_weights(f)
    offs = np.arange(-1, 3)[None, :] - f[:, None]          # node positions minus x, units of h
    np.testing.assert_allclose(w.sum(1), 1.0, atol=1e-14)
    np.testing.assert_allclose((w * offs).sum(1), 0.0, atol=1e-14)
    np.testing.assert_allclose((w * offs ** 2).sum(1), 0.0, atol=1e-14)
    assert np.max(np.abs((w * offs ** 3).sum(1))) > 1e-3   # cubic is not reproduced


def test_keys_continuous_across_cells():
    """f -> 1 in cell j equals f = 0 in cell j+1 (reading A3)."""
    eps = 1e-12
    a = O.keys_weights(np.array([1.0 - eps]))[0]          # nodes j-1..j+2
    b = O.keys_weights(np.array([0.0]))[0]                # nodes j..j+3
    np.testing.assert_allclose(a[1:], b[:3], atol=1e-10)
    assert abs(b[3]) < 1e-15 and abs(a[0]) < 1e-10


def test_interp_node_and_flat_index():
    m, lo, h = (6, 7), (0.0, 10.0), (0.5, 2.0)
    X = np.array([[2 * 0.5, 10.0 + 3 * 2.0]])             # exactly on node (2, 3)
    idx, w = O.interp(X, m, lo, h)
    k = np.argmax(w[0])
    assert w[0, k] == pytest.approx(1.0)
    assert idx[0, k] == 2 * 7 + 3
    assert np.sum(np.abs(w[0])) == pytest.approx(1.0)


def test_interp_out_of_range():
    with pytest.raises(O.OutOfRangeError):
        O.interp_1d(np.array([0.05]), 0.0, 0.1, 10)        # cell 0 needs node -1
    with pytest.raises(O.OutOfRangeError):
        O.interp_1d(np.array([0.85]), 0.0, 0.1, 10)        # cell 8 needs node 10
    O.interp_1d(np.array([0.1, 0.79]), 0.0, 0.1, 10)


def test_W_adjoint_and_dense():
    """<W v, u> == <v, W^T u> and the densified W equals the sparse W."""
    p, inp = tiny_problem("2d")
    idx, w = O.interp(inp.X, p.m, p.lo, p.h)
    rng = np.random.default_rng(1)
    v, u = rng.normal(size=p.n), rng.normal(size=p.m_total)
    Wv = O.W_apply(idx, w, v, p.m_total)
    WTu = O.WT_apply(idx, w, u)
    assert abs(Wv @ u - v @ WTu) < 1e-12 * np.abs(Wv).sum() * np.abs(u).max()
    Wd = O.dense_W(idx, w, p.m_total)
    np.testing.assert_allclose(Wd @ v, Wv, atol=1e-12)
    np.testing.assert_allclose(Wd.T @ u, WTu, atol=1e-12)
    np.testing.assert_allclose(Wd.sum(0), 1.0, atol=1e-13)   # partition of unity per point


# ---------------------------------------------------------------- K_UU
def test_rbf_column_golden():
    for ex in GOLDEN["rbf_column"]:
        np.testing.assert_allclose(O.rbf_column(ex["m"], ex["h"], ex["lengthscale"]),
                                   ex["col"], rtol=1e-15)


def test_toeplitz_golden_dense_and_fft():
    for ex in GOLDEN["toeplitz_mvm"]:
        c, v = np.array(ex["col"], float), np.array(ex["v"], float)
        np.testing.assert_allclose(O.toeplitz_matvec_dense(c, v), ex["out"], atol=1e-14)
        np.testing.assert_allclose(O.toeplitz_matvec_fft(c, v), ex["out"], atol=1e-12)


@pytest.mark.parametrize("m", [1, 2, 7, 64, 1000, 4097])
def test_toeplitz_fft_equals_dense(m):
    rng = np.random.default_rng(m)
    c, v = rng.normal(size=m), rng.normal(size=(m, 3))
    ref = O.toeplitz_dense(c) @ v                        # plain definition
    np.testing.assert_allclose(O.toeplitz_matvec_fft(c, v), ref, atol=1e-10 * np.abs(ref).max())
    np.testing.assert_allclose(O.toeplitz_matvec_dense(c, v), ref, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("m", [(7,), (5, 6), (3, 4, 5)])
def test_kuu_unit_vectors_closed_form(m):
    """K_UU e_q equals the closed form s^2 prod_d exp(-((p_d - q_d) h_d)^2 / (2 l_d^2)) computed
    from grid-node coordinates u = lo + i h (north_star: K_UU entries k(|i-j| h))."""
    d = len(m)
    h = tuple(0.3 + 0.1 * i for i in range(d))
    lo = tuple(-1.0 + i for i in range(d))
    ell = tuple(0.5 + 0.25 * i for i in range(d))
    s2 = 1.7
    cols = [O.rbf_column(m[i], h[i], ell[i]) for i in range(d)]
    M = int(np.prod(m))
    coords = np.stack(np.unravel_index(np.arange(M), m), -1) * np.array(h) + np.array(lo)
    for q in [0, M // 2, M - 1]:
        e = np.zeros(M)
        e[q] = 1.0
        got = O.kuu_matvec(cols, s2, e)
        diff = coords - coords[q]
        want = s2 * np.exp(-0.5 * ((diff / np.array(ell)) ** 2).sum(1))
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-15)


def test_kuu_kronecker_separable_full_size():
    """K_UU (v1 (x) v2 (x) v3) = s^2 (T1 v1) (x) (T2 v2) (x) (T3 v3) at config 4's grid: checks
    the axis/stride logic at full size against 1-D products."""
    p = CONFIGS[4]
    cols = [O.rbf_column(p.m[i], p.h[i], p.lengthscale[i]) for i in range(3)]
    rng = np.random.default_rng(0)
    vs = [rng.normal(size=mm) for mm in p.m]
    v = np.einsum("i,j,k->ijk", *vs).ravel()
    got = O.kuu_matvec(cols, 2.0, v)
    tv = [O.toeplitz_dense(c) @ x for c, x in zip(cols, vs)]
    want = 2.0 * np.einsum("i,j,k->ijk", *tv).ravel()
    np.testing.assert_allclose(got, want, atol=1e-12 * np.abs(want).max())


# ---------------------------------------------------------------- tridiagonal
def test_tridiag_golden():
    for ex in GOLDEN["tridiag_cholesky"]:
        ld, ls = O.tridiag_cholesky(np.array(ex["diag"], float), np.array(ex["off"], float))
        np.testing.assert_allclose(ld, ex["L_diag"])
        np.testing.assert_allclose(ls, ex["L_off"])
    for ex in GOLDEN["tridiag_indefinite"]:
        with pytest.raises(O.NotPDError):
            O.tridiag_cholesky(np.array(ex["diag"], float), np.array(ex["off"], float))
    for ex in GOLDEN["tridiag_solve"]:
        ld, ls = O.tridiag_cholesky(np.array(ex["diag"], float), np.array(ex["off"], float))
        np.testing.assert_allclose(O.tridiag_solve(ld, ls, np.array(ex["b"], float)), ex["x"])


def test_tridiag_random_vs_dense():
    rng = np.random.default_rng(5)
    a = rng.uniform(3, 4, 12)
    b = rng.uniform(-1, 1, 11)
    T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
    ld, ls = O.tridiag_cholesky(a, b)
    L = np.diag(ld) + np.diag(ls, -1)
    np.testing.assert_allclose(L @ L.T, T, atol=1e-13)
    B = rng.normal(size=(12, 3))
    np.testing.assert_allclose(O.tridiag_solve(ld, ls, B), np.linalg.solve(T, B), atol=1e-12)


# ---------------------------------------------------------------- Lanczos
def _spd(n, seed=0, lo=0.1, hi=10.0):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.normal(size=(n, n)))
    ev = np.sort(rng.uniform(lo, hi, n))
    return (U * ev) @ U.T, ev


def test_lanczos_invariants():
    A, ev = _spd(80)
    b = np.random.default_rng(1).normal(size=80)
    lz = O.lanczos(lambda v: A @ v, b, 30)
    Q, T = lz.Q, lz.T
    assert lz.k_eff == 30
    assert np.abs(Q.T @ Q - np.eye(30)).max() < 1e-10               # orthonormal (north_star)
    np.testing.assert_allclose(Q[:, 0], b / np.linalg.norm(b))       # first column = probe
    assert np.all(lz.beta > 0)
    R = A @ Q - Q @ T                                                # A Q_k - Q_k T_k = r e_k^T
    assert np.abs(R[:, :-1]).max() < 1e-10 * ev.max()
    ritz = np.linalg.eigvalsh(T)
    assert ritz.min() >= ev.min() - 1e-8 and ritz.max() <= ev.max() + 1e-8
    np.testing.assert_allclose(Q.T @ A @ Q, T, atol=1e-9)


def test_lanczos_k1_and_identity_breakdown():
    A, _ = _spd(10, seed=2)
    b = np.arange(1.0, 11.0)
    lz = O.lanczos(lambda v: A @ v, b, 1)
    assert lz.alpha[0] == pytest.approx(b @ A @ b / (b @ b), rel=1e-13)
    lz = O.lanczos(lambda v: v.copy(), b, 5)                         # A = I: invariant span{b}
    assert lz.k_eff == 1
    with pytest.raises(O.ZeroProbeError):
        O.lanczos(lambda v: v, np.zeros(4), 3)


def test_lanczos_full_reconstruction_and_solve():
    A, _ = _spd(6, seed=4)
    b = np.random.default_rng(4).normal(size=6)
    lz = O.lanczos(lambda v: A @ v, b, 6)
    np.testing.assert_allclose(lz.Q @ lz.T @ lz.Q.T, A, atol=1e-10)
    for ex in GOLDEN["lanczos_solve"]:                               # Eq. 3
        Ad = np.diag(np.array(ex["A_diag"], float))
        bb = np.array(ex["b"], float)
        lz = O.lanczos(lambda v: Ad @ v, bb, 2)
        ld, ls = O.tridiag_cholesky(lz.alpha, lz.beta)
        e1 = np.eye(lz.k_eff)[0]
        x = np.linalg.norm(bb) * lz.Q @ O.tridiag_solve(ld, ls, e1)
        np.testing.assert_allclose(x, ex["x"], atol=1e-13)
    for ex in GOLDEN["cg_solve"]:
        Ad = np.diag(np.array(ex["A_diag"], float))
        np.testing.assert_allclose(O.cg_solve(lambda v: Ad @ v, np.array(ex["b"], float)),
                                   ex["x"], atol=1e-12)


def test_lanczos_solve_matches_cg_and_dense():
    """Lanczos solve (Eq. 3) and CG agree with a dense solve on an SPD matrix."""
    A, _ = _spd(120, seed=7, lo=1.0, hi=20.0)
    b = np.random.default_rng(7).normal(size=120)
    lz = O.lanczos(lambda v: A @ v, b, 60)
    ld, ls = O.tridiag_cholesky(lz.alpha, lz.beta)
    x = lz.b_norm * lz.Q @ O.tridiag_solve(ld, ls, np.eye(lz.k_eff)[0])
    ref = np.linalg.solve(A, b)
    np.testing.assert_allclose(x, ref, rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(O.cg_solve(lambda v: A @ v, b), ref, rtol=1e-9, atol=1e-10)


# ---------------------------------------------------------------- LOVE (Alg. 1)
@pytest.mark.parametrize("kind", ["1d_n40", "1d_n200", "2d", "3d"])
@pytest.mark.parametrize("probe", ["y", "avg"])
def test_love_equals_dense_ski_gp_at_full_krylov(kind, probe):
    """North_star pin: LOVE run to breakdown (k >= k_eff, 'k = n') reproduces the exact dense
    Cholesky GP with the SKI kernel (Eqs. 1-2, 7) to <= 1e-4 relative (we see ~1e-12)."""
    p, inp = tiny_problem(kind)
    model = _model(p, inp)
    cache = O.love_precompute(model, p.k, probe=probe)
    assert cache.lanczos.k_eff < p.k                                # ran to breakdown
    var = O.predict_var(model, cache, inp.Xs)
    mean = O.predict_mean(model, cache, inp.Xs)
    dmean, dvar = O.dense_ski_gp(model, inp.Xs)
    assert np.max(np.abs(var - dvar) / np.abs(dvar)) < 1e-8
    # probe y: the mean is Eq. 3 for the probe itself (exact at breakdown).  Probe avg: the
    # mean re-uses a Krylov space built for another vector (Eq. 4), only approximately
    # containing y's directions, so it is looser.
    tol = 1e-8 if probe == "y" else 1e-5
    assert np.max(np.abs(mean - dmean)) < tol * np.abs(dmean).max()


def test_love_cfg1_vs_dense_and_cg():
    """Config 1 (fp64, k=50): LOVE vs the dense SKI GP (X1: 5.7e-12) and the mean cache vs a
    CG solve of a = K_UU W_X K_hat^{-1} y."""
    p = CONFIGS[1]
    inp = make_inputs(p)
    model = _model(p, inp)
    cache = O.love_precompute(model, p.k)
    var = O.predict_var(model, cache, inp.Xs)
    dmean, dvar = O.dense_ski_gp(model, inp.Xs)
    assert np.max(np.abs(var - dvar) / dvar) < 1e-6
    sol = O.cg_solve(lambda v: O.ski_mvm(model, v), model.y, tol=1e-13)
    a_cg = O.kuu_matvec(model.cols, model.outputscale, O.W_apply(model.idx, model.w, sol,
                                                                 model.m_total))
    np.testing.assert_allclose(cache.a, a_cg, atol=1e-7 * np.abs(a_cg).max())
    mean = O.predict_mean(model, cache, inp.Xs)
    np.testing.assert_allclose(mean, dmean, atol=1e-7)


def test_love_monotone_in_k_and_bounds():
    """Variance is non-increasing in k (Galerkin over nested Krylov spaces, X10) and lies in
    [0, prior]; covariance is symmetric."""
    p = scaled_config(1, n=400, t=200)
    inp = make_inputs(p)
    model = _model(p, inp)
    prev = None
    for k in [2, 5, 10, 20, 30, 45]:
        cache = O.love_precompute(model, k)
        var = O.predict_var(model, cache, inp.Xs)
        ia, wa = O.interp(inp.Xs, p.m, p.lo, p.h)
        prior = O.prior_ski(model, ia, wa, ia, wa)
        assert np.all(var >= -1e-12) and np.all(var <= prior + 1e-12)
        if prev is not None:
            assert np.all(var <= prev + 1e-10)
        prev = var
    xa, xb = inp.Xs[:50], inp.Xs[50:100]
    np.testing.assert_allclose(O.predict_covar(model, cache, xa, xb),
                               O.predict_covar(model, cache, xb, xa), atol=1e-12)


def test_love_large_noise_limit():
    """sigma^2 -> inf: the posterior variance tends to the prior."""
    p = scaled_config(1, n=300, t=100)
    inp = make_inputs(p)
    model = O.build_model(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, p.outputscale, 1e6)
    cache = O.love_precompute(model, 20)
    var = O.predict_var(model, cache, inp.Xs)
    ia, wa = O.interp(inp.Xs, p.m, p.lo, p.h)
    prior = O.prior_ski(model, ia, wa, ia, wa)
    np.testing.assert_allclose(var, prior, rtol=1e-3)


def test_love_permutation_invariance_and_symmetric_cache():
    """Training order does not change the variances (X2) and R^T R' is symmetric."""
    p = scaled_config(1, n=500, t=100)
    inp = make_inputs(p)
    model = _model(p, inp)
    cache = O.love_precompute(model, 30)
    perm = np.random.default_rng(9).permutation(p.n)
    model2 = O.build_model(inp.X[perm], inp.y[perm], p.m, p.lo, p.h, p.lengthscale,
                           p.outputscale, p.sigma2)
    cache2 = O.love_precompute(model2, 30)
    v1, v2 = O.predict_var(model, cache, inp.Xs), O.predict_var(model2, cache2, inp.Xs)
    np.testing.assert_allclose(v1, v2, rtol=1e-8)
    C = cache.R.T @ cache.Rp
    assert np.abs(C - C.T).max() < 1e-10 * np.abs(C).max()


def test_prior_ski_closed_form():
    """w^T K_UU w from the closed-form entries equals the dense quadratic form."""
    p, inp = tiny_problem("2d")
    model = _model(p, inp)
    ia, wa = O.interp(inp.Xs[:20], p.m, p.lo, p.h)
    Ws = O.dense_W(ia, wa, p.m_total)
    K = O.kuu_dense(model.cols, model.outputscale)
    np.testing.assert_allclose(O.prior_ski(model, ia, wa, ia, wa),
                               np.einsum("it,ij,jt->t", Ws, K, Ws), rtol=1e-13)


def test_prior_exact_vs_library_rbf_and_closed_values():
    """prior_exact (Eq. 10's k(x*_i, x*_j)) at DISTINCT points, pinned three ways
    that share nothing with its own formula:
      * scikit-learn's RBF kernel (exp(-0.5 ||(x - x')/l||^2), anisotropic l) times a
        ConstantKernel(s^2), on random 1-D, 2-D and 3-D pairs;
      * hand values: |x - x'| = l sqrt(2 ln 2) gives s^2 / 2 exactly per dimension (1/8 for three
        such offsets), |x - x'| = l gives s^2 e^{-1/2}; l != 1 so an l-vs-l^2 slip fails;
      * on grid nodes the SKI interpolation is exact, so prior_exact == prior_ski there (the
        latter pinned by K_UU's closed-form entries above)."""
    from sklearn.gaussian_process.kernels import RBF, ConstantKernel
    rng = np.random.default_rng(21)
    for d, ls, s2 in [(1, (0.05,), 1.0), (2, (0.1, 0.3), 2.5), (3, (0.5, 0.7, 1.3), 0.7)]:
        model = types.SimpleNamespace(kind="product", lengthscale=tuple(ls), outputscale=s2)
        Xi = rng.uniform(-1, 1, (200, d))
        Xj = Xi + rng.normal(0, 1, (200, d)) * np.array(ls)          # distinct, O(l) apart
        ref = (ConstantKernel(s2) * RBF(length_scale=np.array(ls)))
        want = np.array([ref(Xi[r:r + 1], Xj[r:r + 1])[0, 0] for r in range(200)])
        np.testing.assert_allclose(O.prior_exact(model, Xi, Xj), want, rtol=1e-13)
        half = np.array(ls) * math.sqrt(2.0 * math.log(2.0))
        got = O.prior_exact(model, np.zeros((1, d)), half[None, :])[0]
        assert abs(got - s2 * 0.5 ** d) < 1e-14 * s2
        one = np.zeros((1, d))
        one[0, 0] = ls[0]
        assert abs(O.prior_exact(model, np.zeros((1, d)), one)[0] - s2 * math.exp(-0.5)) < 1e-14 * s2
    # on grid nodes: exact prior == SKI prior, for distinct node pairs
    p, inp = tiny_problem("2d")
    model = _model(p, inp)
    ni = rng.integers(2, 13, (50, 2))
    nj = rng.integers(2, 13, (50, 2))
    lo, h = np.array(p.lo), np.array(p.h)
    Xi, Xj = lo + ni * h, lo + nj * h
    ia, wa = O.interp(Xi, p.m, p.lo, p.h)
    ib, wb = O.interp(Xj, p.m, p.lo, p.h)
    np.testing.assert_allclose(O.prior_exact(model, Xi, Xj), O.prior_ski(model, ia, wa, ib, wb),
                               rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("kind", ["1d_n200", "2d", "3d"])
def test_predict_covar_offdiagonal_equals_dense_gp(kind):
    """Off-diagonal covariances (Eq. 10) at full Krylov dimension equal the dense
    SKI-GP covariance of Eq. 2, K** - K*X K_hat^{-1} KX*, formed here from the densified W, the
    dense K_UU and a Cholesky solve (no Lanczos), on 400 random pairs of distinct test points;
    the EXACT-prior mode differs from it by exactly k(x_a, x_b) - w_a^T K_UU w_b."""
    p, inp = tiny_problem(kind)
    model = _model(p, inp)
    cache = O.love_precompute(model, p.k)
    assert cache.lanczos.k_eff < p.k
    rng = np.random.default_rng(4)
    a, b = rng.integers(0, p.t, 400), rng.integers(0, p.t, 400)
    keep = a != b
    a, b = a[keep], b[keep]
    Xa, Xb = inp.Xs[a], inp.Xs[b]
    W = O.dense_W(model.idx, model.w, p.m_total)
    Kuu = O.kuu_dense(model.cols, model.outputscale)
    Khat = W.T @ Kuu @ W + p.sigma2 * np.eye(p.n)
    L = np.linalg.cholesky(Khat)
    ia, wa = O.interp(Xa, p.m, p.lo, p.h)
    ib, wb = O.interp(Xb, p.m, p.lo, p.h)
    Wa, Wb = O.dense_W(ia, wa, p.m_total), O.dense_W(ib, wb, p.m_total)
    Ka, Kb = np.linalg.solve(L, W.T @ Kuu @ Wa), np.linalg.solve(L, W.T @ Kuu @ Wb)
    dense = np.einsum("it,ij,jt->t", Wa, Kuu, Wb) - (Ka * Kb).sum(0)
    got = O.predict_covar(model, cache, Xa, Xb)
    scale = np.sqrt(np.abs(O.predict_var(model, cache, Xa) * O.predict_var(model, cache, Xb)))
    assert np.max(np.abs(got - dense) / scale) < 1e-8
    assert np.max(np.abs(O.predict_covar(model, cache, Xb, Xa) - got) / scale) < 1e-10     # symmetry
    ex = O.predict_covar(model, cache, Xa, Xb, prior="exact")
    from sklearn.gaussian_process.kernels import RBF, ConstantKernel
    kab = (ConstantKernel(p.outputscale) * RBF(length_scale=np.array(p.lengthscale)))
    kx = np.array([kab(Xa[r:r + 1], Xb[r:r + 1])[0, 0] for r in range(len(a))])
    np.testing.assert_allclose(ex - got, kx - np.einsum("it,ij,jt->t", Wa, Kuu, Wb), rtol=1e-9, atol=1e-12)


# ---------------------------------------------------------------- sampling
def test_sampling_root_full_rank():
    """With k' >= rank(M), S S^T = K_UU - R^T R', and the implied predictive
    covariance W*^T S S^T W* equals the dense SKI-GP covariance (Eq. 12)."""
    p, inp = tiny_problem("1d_n200")
    model = _model(p, inp)
    cache = O.love_precompute(model, p.k)
    sc = O.sampling_cache(model, cache, 200)
    M = O.kuu_dense(model.cols, model.outputscale) - cache.R.T @ cache.Rp
    assert np.abs(sc.S @ sc.S.T - M).max() < 1e-8 * np.abs(M).max()
    # dense predictive covariance (Eq. 2 with the SKI kernel) at 10 test points
    Xs = inp.Xs[:10]
    ids, ws = O.interp(Xs, p.m, p.lo, p.h)
    Ws = O.dense_W(ids, ws, p.m_total)
    Kuu = O.kuu_dense(model.cols, model.outputscale)
    W = O.dense_W(model.idx, model.w, p.m_total)
    Khat = W.T @ Kuu @ W + p.sigma2 * np.eye(p.n)
    Kxs = W.T @ Kuu @ Ws
    C = Ws.T @ Kuu @ Ws - Kxs.T @ np.linalg.solve(Khat, Kxs)
    G = Ws.T @ sc.S
    assert np.abs(G @ G.T - C).max() < 1e-7 * np.abs(C).max()


def test_sampling_monte_carlo_moments():
    """Sample mean and covariance of mu + W*^T S zeta match mu and W*^T S S^T W* within
    6.5 standard errors (SURVEY §8(c) sampling pin)."""
    p, inp = tiny_problem("1d_n200")
    model = _model(p, inp)
    cache = O.love_precompute(model, p.k)
    sc = O.sampling_cache(model, cache, 60)
    Xs = inp.Xs[:8]
    s = 40000
    zeta = np.random.default_rng(11).normal(size=(sc.lanczos.k_eff, s))
    F = O.draw_samples(model, cache, sc, Xs, zeta)
    mu = O.predict_mean(model, cache, Xs)
    ids, ws = O.interp(Xs, p.m, p.lo, p.h)
    G = np.einsum("tl,tlk->tk", ws, sc.S[ids])
    C = G @ G.T
    Chat = np.cov(F)
    se = np.sqrt((np.outer(np.diag(C), np.diag(C)) + C ** 2) / (s - 1))
    assert np.all(np.abs(Chat - C) <= 6.5 * se)
    assert np.all(np.abs(F.mean(1) - mu) <= 6.5 * np.sqrt(np.diag(C) / s))
    var = O.predict_var(model, cache, Xs)
    np.testing.assert_allclose(np.diag(C), var, rtol=1e-5, atol=1e-10)


def test_smae_definition():
    y = np.array([1.0, 3.0])                                # population variance 1
    assert O.smae(np.array([0.5, 0.5]), np.array([0.0, 1.0]), y) == pytest.approx(0.5)


# ----------------------------------------------------------------- additive kernels (Eq. 16)
def _additive_model(p, inp):
    return O.build_model_additive(inp.X, inp.y, p.m, p.lo, p.h, p.lengthscale, [0.7, 1.3, 1.0][:p.d],
                                  p.sigma2)


def test_additive_kuu_closed_form():
    """Block-diagonal K_UU of Eq. 16: entry (p, q) is s_e^2 exp(-((p-q) h_e)^2 /
    (2 l_e^2)) when p, q are nodes of component e, zero across components."""
    p, inp = tiny_problem("additive3")
    model = _additive_model(p, inp)
    K = O.model_kuu_dense(model)
    s2 = [0.7, 1.3, 1.0]
    off = np.cumsum([0] + list(p.m))
    for a in range(model.m_total):
        for b in range(model.m_total):
            ea = np.searchsorted(off, a, side="right") - 1
            eb = np.searchsorted(off, b, side="right") - 1
            want = 0.0
            if ea == eb:
                want = s2[ea] * math.exp(-((a - b) * p.h[ea]) ** 2 / (2 * p.lengthscale[ea] ** 2))
            assert abs(K[a, b] - want) < 1e-15
    u = np.random.default_rng(3).normal(size=model.m_total)
    np.testing.assert_allclose(O.model_kuu_matvec(model, u), K @ u, rtol=1e-12, atol=1e-12)


def test_additive_kernel_exact_on_nodes():
    """On grid nodes the cubic weights are (0, 1, 0, 0), so the SKI additive kernel
    w_x^T K_UU w_x' equals the exact sum of 1-D kernels (Eq. 16 first line)."""
    p, inp = tiny_problem("additive3")
    model = _additive_model(p, inp)
    rng = np.random.default_rng(5)
    Xa = np.array([[p.lo[e] + rng.integers(2, 12) * p.h[e] for e in range(p.d)] for _ in range(40)])
    Xb = np.array([[p.lo[e] + rng.integers(2, 12) * p.h[e] for e in range(p.d)] for _ in range(40)])
    ia, wa = O.model_interp(model, Xa)
    ib, wb = O.model_interp(model, Xb)
    ski = O.prior_ski(model, ia, wa, ib, wb)
    exact = sum([0.7, 1.3, 1.0][e] * np.exp(-(Xa[:, e] - Xb[:, e]) ** 2 / (2 * p.lengthscale[e] ** 2))
                for e in range(p.d))
    np.testing.assert_allclose(ski, exact, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(O.prior_exact(model, Xa, Xb), exact, rtol=1e-14)


def test_additive_love_equals_dense_gp_at_full_krylov():
    """Eq. 16: Algorithm 1 with the block forms run to breakdown equals the dense
    GP with the additive SKI kernel (Eq. 7 bridge)."""
    p, inp = tiny_problem("additive3")
    model = _additive_model(p, inp)
    cache = O.love_precompute(model, p.k)
    assert cache.lanczos.k_eff < p.k
    mean_d, var_d = O.dense_ski_gp(model, inp.Xs)
    var = O.predict_var(model, cache, inp.Xs)
    np.testing.assert_allclose(var, var_d, rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(O.predict_mean(model, cache, inp.Xs), mean_d, rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("m,ls,span", [(100_000, 0.01, 1.1), (10_000, 0.05, 1.1), (2200, 0.05, 1.1), (300, 0.5, 1.1)])
def test_shortened_circulant_embedding_reading_A25b(m, ls, span):
    """Reading A25b: with b = ceil(ls/h sqrt(2 ln 1e30)) < m, the circulant of
    the smallest power-of-two length N >= m + b reproduces the Toeplitz product to fp64
    rounding.  Checked against the oracle's A25 embedding (N >= 2m - 1) and, at m = 300,
    against the dense Toeplitz matrix; at m = 300 with ls = 0.5 the band is wider than m and
    the rule keeps N >= 2m - 1."""
    h = span / (m - 1)
    c = O.rbf_column(m, h, ls)
    b = int(np.ceil(np.sqrt(2.0 * np.log(1e30)) * ls / h))
    need = min(2 * m - 1, m + b) if b < m else 2 * m - 1
    N = 8
    while N < need:
        N *= 2
    if m == 100_000:
        assert N == 1 << 17                      # cfg2: half of A25's 2^18
    a = np.minimum(np.arange(N), N - np.arange(N))
    col = np.where(a < m, c[np.minimum(a, m - 1)], 0.0)
    if b < m:                                    # b is where the column falls below 1e-30 c_0
        assert c[b] < 1e-30 * c[0] <= c[b - 1]
    u = np.random.default_rng(3).normal(size=(m, 2))
    got = np.fft.ifft(np.fft.fft(col)[:, None] * np.fft.fft(np.vstack([u, np.zeros((N - m, 2))]), axis=0),
                      axis=0)[:m].real
    want = O.toeplitz_matvec_dense(c, u) if m <= 2200 else O.toeplitz_matvec_fft(c, u)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
