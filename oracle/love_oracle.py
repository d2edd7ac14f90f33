"""LOVE (LanczOs Variance Estimates) for KISS-GP -- plain fp64 CPU oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain, slow, obviously correct numpy:
no blocking, fusion or reordering beyond what the paper's equations and Algorithm 1 state.
Library primitives used as single steps: numpy FFT (circulant product), matmul/gemv,
bincount (a sparse sum), Cholesky / triangular solves / symmetric eigendecomposition of
small dense matrices.

Citations: P:<n> = /root/reference/PAPER.md line n; S:<n> = SPEC.md line n (interfaces and
test ideas only); A<n> = reading n of SURVEY.md §8(c) (also listed in DESIGN.md).

Pins (tests/test_oracle_pins.py, all `-m "not gpu"`):
  keys_kernel / interp_1d / interp ......... closed-form Keys values, polynomial reproduction,
                                              densified-W adjointness            -> pinned
  rbf_column / kuu_matvec .................. closed-form K_UU[i,j] entries on unit vectors,
                                              Kronecker separability, FFT == dense -> pinned
  lanczos .................................. QtQ = I, three-term relation, Ritz containment,
                                              A = I breakdown, full-rank reconstruction,
                                              Lanczos solve == dense solve          -> pinned
  tridiag_cholesky / tridiag_solve ......... hand-derived 2x2 examples, indefinite error -> pinned
  love_precompute / predict_var / covar .... == dense-Cholesky SKI GP at full Krylov
                                              dimension; monotone in k; 0 <= var <= prior -> pinned
  mean cache ............................... == dense SKI GP mean; == CG solve      -> pinned
  sampling_cache / draw_samples ............ SS^T == K_UU - R^T R' at full rank; Monte-Carlo
                                              moments                                -> pinned
  additive models (Eq. 16) ....... block-diagonal K_UU == sum of 1-D kernels on
                                              node pairs; stacked W adjointness; LOVE ==
                                              dense SKI GP of the additive kernel at full
                                              Krylov dimension                       -> pinned
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "OracleError", "OutOfRangeError", "ZeroProbeError", "NotPDError",
    "keys_kernel", "keys_weights", "interp_1d", "interp", "dense_W",
    "rbf_column", "toeplitz_dense", "toeplitz_matvec_dense", "toeplitz_matvec_fft",
    "kuu_matvec", "kuu_dense", "SKIModel", "build_model", "W_apply", "WT_apply", "ski_mvm",
    "lanczos", "LanczosResult", "tridiag_cholesky", "tridiag_solve",
    "LoveCache", "love_precompute", "prior_ski", "prior_exact", "predict_mean",
    "predict_var", "predict_covar", "sampling_cache", "draw_samples", "SamplingCache",
    "dense_ski_gp", "cg_solve", "smae",
    "build_model_additive", "interp_additive", "model_interp", "model_kuu_matvec", "model_kuu_dense",
]


class OracleError(RuntimeError):
    pass


class OutOfRangeError(OracleError):
    """A point needs a grid node outside [0, m_d - 1] (reading A4)."""


class ZeroProbeError(OracleError):
    """Lanczos probe b = 0."""


class NotPDError(OracleError):
    """A pivot of the tridiagonal Cholesky is <= 0 (reading A13)."""


# --------------------------------------------------------------------------------------
# Cubic-convolution interpolation (SKI; Keys cubic with a = -1/2, reading A2)
# --------------------------------------------------------------------------------------
KEYS_A = -0.5


def keys_kernel(s: np.ndarray, a: float = KEYS_A) -> np.ndarray:
    """Keys' cubic convolution kernel u(s) (P:177 cites keys1981cubic):
         (a+2)|s|^3 - (a+3)|s|^2 + 1        |s| <= 1
         a|s|^3 - 5a|s|^2 + 8a|s| - 4a      1 < |s| < 2
         0                                  otherwise"""
    s = np.abs(np.asarray(s, dtype=np.float64))
    out = np.zeros_like(s)
    near = s <= 1.0
    far = (s > 1.0) & (s < 2.0)
    out[near] = (a + 2.0) * s[near] ** 3 - (a + 3.0) * s[near] ** 2 + 1.0
    out[far] = a * s[far] ** 3 - 5.0 * a * s[far] ** 2 + 8.0 * a * s[far] - 4.0 * a
    return out


def keys_weights(f: np.ndarray) -> np.ndarray:
    """Weights of the 4 closest nodes j-1, j, j+1, j+2 of a point at u_j + f*h, 0 <= f < 1
    ("its 4 closest inducing points"): u(1+f), u(f), u(1-f), u(2-f).  Shape (..., 4)."""
    f = np.asarray(f, dtype=np.float64)
    return np.stack([keys_kernel(1.0 + f), keys_kernel(f), keys_kernel(1.0 - f),
                     keys_kernel(2.0 - f)], axis=-1)


def interp_1d(x: np.ndarray, lo: float, h: float, m: int) -> Tuple[np.ndarray, np.ndarray]:
    """Indices (n,4) and weights (n,4) of 1-D cubic interpolation on u_i = lo + i*h.
    Cell j = floor((x-lo)/h) in fp64, frac f = (x-lo)/h - j (reading A3); the stencil
    j-1..j+2 must lie in [0, m-1], i.e. 1 <= j <= m-3 (reading A4), else OutOfRangeError."""
    x = np.asarray(x, dtype=np.float64)
    s = (x - lo) / h
    j = np.floor(s)
    f = s - j
    j = j.astype(np.int64)
    bad = (j < 1) | (j > m - 3)
    if np.any(bad):
        raise OutOfRangeError(f"{int(bad.sum())} point(s) outside the interpolable grid")
    idx = j[:, None] - 1 + np.arange(4)[None, :]
    return idx, keys_weights(f)


def interp(X: np.ndarray, m: Sequence[int], lo: Sequence[float], h: Sequence[float]
           ) -> Tuple[np.ndarray, np.ndarray]:
    """Interpolation vectors w_x for a d-dimensional grid (Kronecker grid):
    the tensor product of the per-dimension 4-point stencils, 4^d nonzeros per point.
    Flat node index is row-major (last dimension fastest).  Returns idx, w of shape (n, 4^d),
    slot order row-major in (l_1, ..., l_d)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    n, d = X.shape
    idx = np.zeros((n, 1), dtype=np.int64)
    w = np.ones((n, 1), dtype=np.float64)
    for dim in range(d):
        i_d, w_d = interp_1d(X[:, dim], lo[dim], h[dim], m[dim])
        idx = (idx[:, :, None] * m[dim] + i_d[:, None, :]).reshape(n, -1)
        w = (w[:, :, None] * w_d[:, None, :]).reshape(n, -1)
    return idx, w


def dense_W(idx: np.ndarray, w: np.ndarray, m_total: int) -> np.ndarray:
    """W_X as a dense m x n matrix, columns w_{x_i}."""
    n = idx.shape[0]
    W = np.zeros((m_total, n))
    np.add.at(W, (idx, np.repeat(np.arange(n)[:, None], idx.shape[1], 1)), w)
    return W


# --------------------------------------------------------------------------------------
# K_UU on a regular grid: Toeplitz (1-D) / Kronecker of Toeplitz (d-D)
# --------------------------------------------------------------------------------------
def rbf_column(m_d: int, h_d: float, lengthscale: float) -> np.ndarray:
    """First column of the 1-D RBF kernel matrix on the grid: c[i] = exp(-(i h)^2 / (2 l^2))
    (reading A6: k(r) = s^2 exp(-r^2/(2 l^2)); the s^2 is applied once in
    kuu_matvec)."""
    r = np.arange(m_d, dtype=np.float64) * h_d
    return np.exp(-(r * r) / (2.0 * lengthscale * lengthscale))


def toeplitz_dense(c: np.ndarray) -> np.ndarray:
    """Symmetric Toeplitz matrix T[i,j] = c[|i-j|] ("Toeplitz structure")."""
    m = len(c)
    i = np.arange(m)
    return c[np.abs(i[:, None] - i[None, :])]


def toeplitz_matvec_dense(c: np.ndarray, V: np.ndarray) -> np.ndarray:
    """T(c) @ V by forming T densely (plain definition)."""
    return toeplitz_dense(c) @ V


def toeplitz_matvec_fft(c: np.ndarray, V: np.ndarray) -> np.ndarray:
    """T(c) @ V through the circulant embedding of length N = 2^ceil(log2(2m-1)) (reading
    A25; "MVMs in at most O(n + m log m)"; numpy FFT as the library step):
    col = [c_0..c_{m-1}, 0, .., 0, c_{m-1}..c_1], T v = first m of IFFT(FFT(col) * FFT([v;0]))."""
    m = len(c)
    N = 1
    while N < 2 * m - 1:
        N *= 2
    col = np.zeros(N)
    col[:m] = c
    if m > 1:
        col[N - m + 1:] = c[1:][::-1]
    lam = np.fft.fft(col)
    V2 = V.reshape(m, -1)
    pad = np.zeros((N, V2.shape[1]))
    pad[:m] = V2
    out = np.fft.ifft(lam[:, None] * np.fft.fft(pad, axis=0), axis=0)[:m].real
    return out.reshape(V.shape)


DENSE_TOEPLITZ_MAX = 4096


def _toeplitz_apply(c: np.ndarray, V: np.ndarray) -> np.ndarray:
    if len(c) <= DENSE_TOEPLITZ_MAX:
        return toeplitz_matvec_dense(c, V)
    return toeplitz_matvec_fft(c, V)


def kuu_matvec(cols: Sequence[np.ndarray], outputscale: float, u: np.ndarray) -> np.ndarray:
    """K_UU u with K_UU = s^2 * T(c_1) (x) ... (x) T(c_d) (Kronecker of Toeplitz):
    apply T(c_dim) along axis `dim` of u reshaped to (m_1, ..., m_d).  Works on a batch of
    vectors u of shape (m_total,) or (m_total, b)."""
    shape = tuple(len(c) for c in cols)
    batch = u.shape[1:] if u.ndim > 1 else ()
    U = u.reshape(shape + batch)
    for dim, c in enumerate(cols):
        U = np.moveaxis(U, dim, 0)
        moved = U.shape
        U = _toeplitz_apply(c, U.reshape(moved[0], -1)).reshape(moved)
        U = np.moveaxis(U, 0, dim)
    return outputscale * U.reshape(u.shape)


def kuu_dense(cols: Sequence[np.ndarray], outputscale: float) -> np.ndarray:
    """Dense K_UU = s^2 * kron(T(c_1), ..., T(c_d)) (tiny grids only)."""
    K = np.ones((1, 1))
    for c in cols:
        K = np.kron(K, toeplitz_dense(c))
    return outputscale * K


# --------------------------------------------------------------------------------------
# The SKI operator  K_hat = W_X^T K_UU W_X + sigma^2 I
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class SKIModel:
    m: Tuple[int, ...]
    lo: Tuple[float, ...]
    h: Tuple[float, ...]
    cols: List[np.ndarray]
    outputscale: float
    lengthscale: Tuple[float, ...]
    sigma2: float
    idx: np.ndarray           # (n, 4^d) training stencils  (additive: (n, 4d))
    w: np.ndarray             # (n, 4^d) training weights
    y: np.ndarray             # (n,)
    kind: str = "product"     # "product" (Kronecker grid) | "additive" (Eq. 16)
    outputscales: Tuple[float, ...] = ()   # additive: per-component s_e^2

    @property
    def m_total(self) -> int:
        return int(np.sum(self.m)) if self.kind == "additive" else int(np.prod(self.m))

    @property
    def offsets(self) -> np.ndarray:
        """additive: first node of component e in the stacked inducing set"""
        return np.concatenate([[0], np.cumsum(self.m)[:-1]]).astype(np.int64)

    @property
    def n(self) -> int:
        return self.idx.shape[0]


def build_model(X, y, m, lo, h, lengthscale, outputscale, sigma2) -> SKIModel:
    m = tuple(int(v) for v in m)
    cols = [rbf_column(m[i], h[i], lengthscale[i]) for i in range(len(m))]
    idx, w = interp(X, m, lo, h)
    return SKIModel(m, tuple(lo), tuple(h), cols, float(outputscale), tuple(lengthscale),
                    float(sigma2), idx, w, np.asarray(y, dtype=np.float64))


# --------------------------------------------------------------------------------------
# Additive compositions (Eq. 16): k~(x, x') = sum_e w^(e)_x^T K^(e)_UU w^(e)_x',
# i.e. stacked interpolation vectors [w^(1); ..; w^(d)] (4 nonzeros per component, 4d per
# point) and a block-diagonal K_UU = diag(K^(1), .., K^(d)) of 1-D Toeplitz blocks.
# --------------------------------------------------------------------------------------
def interp_additive(X: np.ndarray, m: Sequence[int], lo: Sequence[float], h: Sequence[float]
                    ) -> Tuple[np.ndarray, np.ndarray]:
    """Stacked block interpolation vectors of Eq. 16: component e contributes its 1-D cubic
    stencil on its own grid, at node offset sum_{e' < e} m_e'.  Returns (n, 4d)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X[:, None]
    off = 0
    idxs, ws = [], []
    for e in range(X.shape[1]):
        i_e, w_e = interp_1d(X[:, e], lo[e], h[e], m[e])
        idxs.append(i_e + off)
        ws.append(w_e)
        off += int(m[e])
    return np.concatenate(idxs, axis=1), np.concatenate(ws, axis=1)


def build_model_additive(X, y, m, lo, h, lengthscale, outputscales, sigma2) -> SKIModel:
    """SKI model of the additive kernel sum_e s_e^2 exp(-(x_e - x'_e)^2 / (2 l_e^2)) (Eq. 16;
    RBF components as in the paper's Styblinski-Tang model)."""
    m = tuple(int(v) for v in m)
    cols = [rbf_column(m[i], h[i], lengthscale[i]) for i in range(len(m))]
    idx, w = interp_additive(X, m, lo, h)
    return SKIModel(m, tuple(lo), tuple(h), cols, 1.0, tuple(lengthscale), float(sigma2), idx, w,
                    np.asarray(y, dtype=np.float64), kind="additive",
                    outputscales=tuple(float(v) for v in outputscales))


def model_interp(model: SKIModel, X: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Interpolation vectors of test points for the model's structure."""
    if model.kind == "additive":
        return interp_additive(X, model.m, model.lo, model.h)
    return interp(X, model.m, model.lo, model.h)


def model_kuu_matvec(model: SKIModel, u: np.ndarray) -> np.ndarray:
    """K_UU u: Kronecker of Toeplitz, or the block-diagonal K_UU of Eq. 16 (each block
    s_e^2 T(c_e) applied to its slice)."""
    if model.kind != "additive":
        return kuu_matvec(model.cols, model.outputscale, u)
    out = np.zeros_like(u, dtype=np.float64)
    off = 0
    for e, c in enumerate(model.cols):
        sl = slice(off, off + len(c))
        out[sl] = model.outputscales[e] * _toeplitz_apply(c, u[sl].reshape(len(c), -1)).reshape(u[sl].shape)
        off += len(c)
    return out


def model_kuu_dense(model: SKIModel) -> np.ndarray:
    if model.kind != "additive":
        return kuu_dense(model.cols, model.outputscale)
    M = model.m_total
    K = np.zeros((M, M))
    off = 0
    for e, c in enumerate(model.cols):
        K[off:off + len(c), off:off + len(c)] = model.outputscales[e] * toeplitz_dense(c)
        off += len(c)
    return K


def W_apply(idx: np.ndarray, w: np.ndarray, v: np.ndarray, m_total: int) -> np.ndarray:
    """u = W_X v (n -> m): u[idx_l] += w_l v_i over all points and stencil slots."""
    return np.bincount(idx.ravel(), weights=(w * v[:, None]).ravel(), minlength=m_total)


def WT_apply(idx: np.ndarray, w: np.ndarray, z: np.ndarray) -> np.ndarray:
    """g = W_X^T z (m -> n): g_i = w_{x_i}^T z."""
    return (w * z[idx]).sum(axis=1)


def ski_mvm(model: SKIModel, v: np.ndarray) -> np.ndarray:
    """(W_X^T K_UU W_X + sigma^2 I) v  (Eq. 5 P:180 plus noise, mvm_K_XX of Alg. 1)."""
    u = W_apply(model.idx, model.w, v, model.m_total)
    z = model_kuu_matvec(model, u)
    return WT_apply(model.idx, model.w, z) + model.sigma2 * v


# --------------------------------------------------------------------------------------
# Lanczos tridiagonalisation with full reorthogonalisation
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class LanczosResult:
    Q: np.ndarray             # (n, k_eff), orthonormal columns
    alpha: np.ndarray         # (k_eff,) diagonal of T
    beta: np.ndarray          # (k_eff-1,) off-diagonal of T
    k_eff: int
    b_norm: float

    @property
    def T(self) -> np.ndarray:
        return np.diag(self.alpha) + np.diag(self.beta, 1) + np.diag(self.beta, -1)


def lanczos(matvec, b: np.ndarray, k: int, tau: float = 1e-10, reorth_passes: int = 2
            ) -> LanczosResult:
    """k steps of Lanczos on the symmetric operator `matvec` from probe b:
        q_1 = b/||b||, beta_0 = 0; for j = 1..k:
          v = A q_j; alpha_j = q_j^T v; v -= alpha_j q_j + beta_{j-1} q_{j-1}
          full reorthogonalisation, twice: v -= Q_j (Q_j^T v)   (reading A10: CGS2)
          beta_j = ||v||; breakdown if beta_j < tau (max|alpha| + 2 max beta)  (reading A12)
          q_{j+1} = v / beta_j
    T bookkeeping holds the recurrence alpha_j and the norms beta_j (reading A11)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    b_norm = float(np.linalg.norm(b))
    if b_norm == 0.0:
        raise ZeroProbeError("zero probe vector")
    k = min(int(k), n)
    Q = np.zeros((n, k), order="F")
    alpha: List[float] = []
    beta: List[float] = []
    Q[:, 0] = b / b_norm
    k_eff = k
    for j in range(k):
        v = matvec(Q[:, j])
        a = float(Q[:, j] @ v)
        alpha.append(a)
        if j == k - 1:
            break
        v = v - a * Q[:, j]
        if j > 0:
            v = v - beta[j - 1] * Q[:, j - 1]
        for _ in range(reorth_passes):
            Qj = Q[:, :j + 1]
            v = v - Qj @ (Qj.T @ v)
        bj = float(np.linalg.norm(v))
        anorm = max(abs(x) for x in alpha) + 2.0 * max(beta + [bj])
        if bj < tau * anorm:
            k_eff = j + 1
            break
        beta.append(bj)
        Q[:, j + 1] = v / bj
    return LanczosResult(Q[:, :k_eff].copy(order="F"), np.array(alpha[:k_eff]),
                         np.array(beta[:k_eff - 1]), k_eff, b_norm)


def tridiag_cholesky(alpha: np.ndarray, beta: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """T = L L^T with L lower bidiagonal (O(k)):
    L_11 = sqrt(alpha_1); L_{j,j-1} = beta_{j-1} / L_{j-1,j-1}; L_jj = sqrt(alpha_j - L_{j,j-1}^2).
    A pivot <= 0 raises NotPDError (reading A13)."""
    k = len(alpha)
    ld = np.zeros(k)
    ls = np.zeros(max(k - 1, 0))
    for j in range(k):
        piv = alpha[j] - (ls[j - 1] ** 2 if j > 0 else 0.0)
        if not piv > 0.0:
            raise NotPDError(f"tridiagonal Cholesky pivot {piv} at {j}")
        ld[j] = math.sqrt(piv)
        if j < k - 1:
            ls[j] = beta[j] / ld[j]
    return ld, ls


def tridiag_solve(ld: np.ndarray, ls: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Solve (L L^T) X = B with the bidiagonal factor: forward then backward substitution
    ("compute T^{-1} R^T using the Cholesky decomposition of T")."""
    B = np.array(B, dtype=np.float64, copy=True)
    k = len(ld)
    Y = np.zeros_like(B)
    for j in range(k):
        acc = B[j] - (ls[j - 1] * Y[j - 1] if j > 0 else 0.0)
        Y[j] = acc / ld[j]
    Xs = np.zeros_like(B)
    for j in range(k - 1, -1, -1):
        acc = Y[j] - (ls[j] * Xs[j + 1] if j < k - 1 else 0.0)
        Xs[j] = acc / ld[j]
    return Xs


# --------------------------------------------------------------------------------------
# LOVE pre-computation, Algorithm 1, paper-literal R and R'
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class LoveCache:
    R: np.ndarray             # (k, m)  R  = (K_UU W_X Q_k)^T
    Rp: np.ndarray            # (k, m)  R' = T_k^{-1} R
    a: np.ndarray             # (m,)    mean cache
    lanczos: LanczosResult
    Ld: np.ndarray
    Ls: np.ndarray
    probe: str


def love_precompute(model: SKIModel, k: int, probe: str = "y", tau: float = 1e-10,
                    reorth_passes: int = 2) -> LoveCache:
    """Algorithm 1, lines P:391-399:
        Q_k, T_k <- lanczos_k(mvm_K_XX, b)
        L_{T_k} <- cholesky_factor(T_k)
        R  <- (mvm_K_UX(Q_k))^T          (k fresh scatters W_X q_i and K_UU MVMs)
        R' <- cholesky_solve(R, L_{T_k})
    Probe (reading A1): 'y' (default: the training targets, so the mean cache follows from
    Eq. 3) or 'avg' (b = (1/m) W_X^T K_UU 1, P:286 / P:386).
    Mean cache a = K_UU W_X K_hat^{-1} y (Eq. 6): probe y -> ||y|| R^T T^{-1} e_1
    (Eq. 3); probe avg -> R^T T^{-1} Q^T y (Eq. 4)."""
    if probe == "y":
        b = model.y
    elif probe == "avg":
        ones = np.ones(model.m_total)
        b = WT_apply(model.idx, model.w, model_kuu_matvec(model, ones))
        b = b / model.m_total
    else:
        raise ValueError(probe)
    lz = lanczos(lambda v: ski_mvm(model, v), b, k, tau=tau, reorth_passes=reorth_passes)
    Ld, Ls = tridiag_cholesky(lz.alpha, lz.beta)
    kk = lz.k_eff
    R = np.zeros((kk, model.m_total))
    for i in range(kk):                      # mvm_K_UX(q_i) = K_UU (W_X q_i)
        u = W_apply(model.idx, model.w, lz.Q[:, i], model.m_total)
        R[i] = model_kuu_matvec(model, u)
    Rp = tridiag_solve(Ld, Ls, R)
    if probe == "y":
        e1 = np.zeros(kk)
        e1[0] = 1.0
        a = lz.b_norm * (R.T @ tridiag_solve(Ld, Ls, e1))
    else:
        a = R.T @ tridiag_solve(Ld, Ls, lz.Q.T @ model.y)
    return LoveCache(R, Rp, a, lz, Ld, Ls, probe)


def prior_ski(model: SKIModel, idx_i, w_i, idx_j, w_j) -> np.ndarray:
    """SKI prior covariance w_i^T K_UU w_j (Eq. 12 first term; reading A8), one value
    per pair (row i of the test set with row j), computed from closed-form K_UU entries
    K_UU[p,q] = s^2 prod_d c_d[|p_d - q_d|]."""
    t = idx_i.shape[0]
    out = np.zeros(t)
    if model.kind == "additive":
        # K_UU[p, q] = s_e^2 c_e[|p - q|] when p, q are nodes of the same component e, else 0
        off = model.offsets
        comp_i = np.searchsorted(off, idx_i, side="right") - 1
        comp_j = np.searchsorted(off, idx_j, side="right") - 1
        for a in range(idx_i.shape[1]):
            for b in range(idx_j.shape[1]):
                same = comp_i[:, a] == comp_j[:, b]
                e = comp_i[:, a]
                kv = np.zeros(t)
                for ee in np.unique(e[same]):
                    sel = same & (e == ee)
                    kv[sel] = model.outputscales[ee] * model.cols[ee][np.abs(idx_i[sel, a] - idx_j[sel, b])]
                out += w_i[:, a] * w_j[:, b] * kv
        return out
    coords_i = np.stack(np.unravel_index(idx_i, model.m), axis=-1)   # (t, 4^d, d)
    coords_j = np.stack(np.unravel_index(idx_j, model.m), axis=-1)
    for a in range(idx_i.shape[1]):
        for b in range(idx_j.shape[1]):
            kv = np.ones(t)
            for d, c in enumerate(model.cols):
                kv = kv * c[np.abs(coords_i[:, a, d] - coords_j[:, b, d])]
            out += w_i[:, a] * w_j[:, b] * kv
    return model.outputscale * out


def _as2d(X: np.ndarray) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    return X[:, None] if X.ndim == 1 else X


def prior_exact(model: SKIModel, Xi: np.ndarray, Xj: np.ndarray) -> np.ndarray:
    """Exact prior k(x_i, x_j) = s^2 prod_d exp(-(x_id - x_jd)^2 / (2 l_d^2)) (Eq. 10)."""
    Xi, Xj = _as2d(Xi), _as2d(Xj)
    if model.kind == "additive":          # sum_e s_e^2 exp(-(x_e - x'_e)^2 / (2 l_e^2))  (Eq. 16)
        out = np.zeros(Xi.shape[0])
        for e, l in enumerate(model.lengthscale):
            out += model.outputscales[e] * np.exp(-0.5 * (Xi[:, e] - Xj[:, e]) ** 2 / (l * l))
        return out
    r2 = np.zeros(Xi.shape[0])
    for d, l in enumerate(model.lengthscale):
        r2 += (Xi[:, d] - Xj[:, d]) ** 2 / (l * l)
    return model.outputscale * np.exp(-0.5 * r2)


def predict_mean(model: SKIModel, cache: LoveCache, Xs: np.ndarray) -> np.ndarray:
    """mu(x*) = w_{x*}^T a (Eq. 6; zero prior mean, reading A19)."""
    idx, w = model_interp(model, Xs)
    return (w * cache.a[idx]).sum(1)


def predict_covar(model: SKIModel, cache: LoveCache, Xa: np.ndarray, Xb: np.ndarray,
                  prior: str = "ski") -> np.ndarray:
    """k(x*_i, x*_j) ~= k_{x*_i x*_j} - (R w*_i)^T R' w*_j  (Eq. 10; Alg. 1
    P:401-403: u = sparse_mm(R, w_i), v = sparse_mm(R', w_j), return k_ij - u^T v).
    One value per row pair (Xa[r], Xb[r])."""
    Xa, Xb = _as2d(Xa), _as2d(Xb)
    out = np.zeros(Xa.shape[0])
    for s in range(0, Xa.shape[0], 16384):                   # chunked only to bound memory
        e = min(s + 16384, Xa.shape[0])
        ia, wa = model_interp(model, Xa[s:e])
        ib, wb = model_interp(model, Xb[s:e])
        u = np.einsum("tl,ktl->tk", wa, cache.R[:, ia])       # R w_i   (t, k)
        v = np.einsum("tl,ktl->tk", wb, cache.Rp[:, ib])      # R' w_j  (t, k)
        if prior == "ski":
            p = prior_ski(model, ia, wa, ib, wb)
        elif prior == "exact":
            p = prior_exact(model, Xa[s:e], Xb[s:e])
        else:
            raise ValueError(prior)
        out[s:e] = p - (u * v).sum(1)
    return out


def predict_var(model: SKIModel, cache: LoveCache, Xs: np.ndarray, prior: str = "ski"
                ) -> np.ndarray:
    """Predictive variance: Eq. 10 with x*_i = x*_j (O(k) per query)."""
    return predict_covar(model, cache, Xs, Xs, prior)


# --------------------------------------------------------------------------------------
# Sampling (Eqs. 11-15)
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class SamplingCache:
    S: np.ndarray             # (m, k') root with S S^T ~= K_UU - R^T R'
    lanczos: LanczosResult
    evals: np.ndarray         # eigenvalues of T' before clamping


def sampling_cache(model: SKIModel, cache: LoveCache, k_sample: int, tau: float = 1e-10
                   ) -> SamplingCache:
    """Lanczos on M = K_UU - R^T R' (Eq. 12-13), k' steps from probe M 1
    (reading A14), then the root of T'_k: reading A15 replaces the Cholesky of T'
    (singular at breakdown) by the clamped symmetric root T'^{1/2} = V max(L,0)^{1/2} V^T,
    S = Q' T'^{1/2} (P:357 with L_{T_k} read as the root of T'_k, reading A18), so that
    S S^T = Q' T' Q'^T (Eq. 14-15)."""
    def mvm(v):
        return model_kuu_matvec(model, v) - cache.R.T @ (cache.Rp @ v)

    b = mvm(np.ones(model.m_total))
    lz = lanczos(mvm, b, k_sample, tau=tau, reorth_passes=2)
    evals, V = np.linalg.eigh(lz.T)
    root = (V * np.sqrt(np.maximum(evals, 0.0))[None, :]) @ V.T
    return SamplingCache(lz.Q @ root, lz, evals)


def draw_samples(model: SKIModel, cache: LoveCache, scache: SamplingCache, Xs: np.ndarray,
                 zeta: np.ndarray) -> np.ndarray:
    """Posterior samples mu(X*) + W_{X*}^T S zeta (Eq. 11).
    zeta: (k'_eff, s) standard normals (columns = samples).  Returns (t, s)."""
    idx, w = model_interp(model, Xs)
    mu = (w * cache.a[idx]).sum(1)
    G = np.einsum("tl,tlk->tk", w, scache.S[idx])          # W_{X*}^T S   (t, k')
    return mu[:, None] + G @ zeta


# --------------------------------------------------------------------------------------
# Dense bridge (tiny inputs): exact GP with the SKI kernel, Eqs. 1-2 / 7
# --------------------------------------------------------------------------------------
def dense_ski_gp(model: SKIModel, Xs: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Predictive mean and variance of the GP whose kernel is the SKI kernel
    k~(x, x') = w_x^T K_UU w_x' (Eq. 5), by dense Cholesky of
    K_hat = W_X^T K_UU W_X + sigma^2 I:
        mu = k~_{X x*}^T K_hat^{-1} y,  var = w*^T K_UU w* - k~^T K_hat^{-1} k~  (Eq. 7)."""
    Kuu = model_kuu_dense(model)
    W = dense_W(model.idx, model.w, model.m_total)          # m x n
    Khat = W.T @ Kuu @ W + model.sigma2 * np.eye(model.n)
    L = np.linalg.cholesky(Khat)
    ids, ws = model_interp(model, Xs)
    Ws = dense_W(ids, ws, model.m_total)                    # m x t
    Kxs = W.T @ Kuu @ Ws                                    # n x t
    alpha = np.linalg.solve(L.T, np.linalg.solve(L, model.y))
    mean = Kxs.T @ alpha
    V = np.linalg.solve(L, Kxs)
    var = np.einsum("it,ij,jt->t", Ws, Kuu, Ws) - (V * V).sum(0)
    return mean, var


def cg_solve(matvec, b: np.ndarray, tol: float = 1e-12, max_iter: int = 10000) -> np.ndarray:
    """Linear conjugate gradients: the three-term recurrence minimising
    1/2 x^T A x - x^T b, one MVM per iteration."""
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = float(r @ r)
    bn = math.sqrt(float(b @ b))
    for _ in range(max_iter):
        if math.sqrt(rr) <= tol * bn:
            break
        Ap = matvec(p)
        step = rr / float(p @ Ap)
        x += step * p
        r -= step * Ap
        rr_new = float(r @ r)
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x


def smae(pred: np.ndarray, ref: np.ndarray, y: np.ndarray) -> float:
    """Standardised mean absolute error: MAE divided by the (population) variance of the
    training targets (reading A22)."""
    return float(np.mean(np.abs(pred - ref)) / np.var(y))
