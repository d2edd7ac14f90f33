// sample.cu -- posterior sampling with LOVE (Eqs. 11-15).
//
// Sampling cache (build time, fp64, reading A16):
//   M v = K_UU v - Rc (Rc^T v)            (Eq. 12 / 13: K_UU - R^T R', Rc Rc^T = R^T R')
//   k' Lanczos steps on M from b' = M 1 (reading A14), three-term + CGS2,
//   breakdown rule of reading A12  ->  Q' (m x k'), T' (k' x k'); the steps run on the grid
//   Lanczos machinery (device step index, CUDA-graph replay, the fp64 reorthogonalisation
//   kernels of lanczos.cu) with this operator and without the Cholesky of T
//   T' = V diag(lambda) V^T (multisection + twisted factorisation, one CTA), T'^{1/2} = V diag(sqrt(max(lambda, 0))) V^T
//   S = Q' T'^{1/2}  (reading A15: the unique PSD root replaces the Cholesky factor of P:351)
// Draws (love_sample):
//   G = W_{X*}^T S (t x k'),  mu = W_{X*}^T a,  F = mu 1^T + G zeta    (Eq. 11)
//   zeta from the caller (shared-draw parity) or Philox4x32-10 + Box-Muller (reading A24).
#include <cuda_runtime.h>
#include <type_traits>
#include <cstdlib>

#include <cmath>

#include "love_internal.h"
#include "ski_device.cuh"

namespace love {

LOVE_TRACE_TU(sample)

namespace {

constexpr int kMaxKs = 112;          // k' limit of the single-CTA Jacobi eigensolver (smem)

// out[c] += sum_r A[r + c*lda] * x[r], c < ncol   (fp64, CTA row tiles, warps own columns)
constexpr int kDotRows = 64;        // rows per CTA tile of dots_kernel (~m/64 CTAs)
__global__ void __launch_bounds__(256) dots_kernel(const double* __restrict__ A, int64_t lda, int nrow, int ncol,
                                                   const double* __restrict__ x, double* __restrict__ out,
                                                   const int* __restrict__ stop) {
    pdl_wait();
    if (stop && *stop) return;
    __shared__ double xs[kDotRows];
    const int r0 = blockIdx.x * kDotRows;
    const int nr = min(kDotRows, nrow - r0);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) xs[i] = x[r0 + i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c = wid; c < ncol; c += nw) {
        const double* a = A + (int64_t)c * lda + r0;
        double acc = 0.0;
        for (int i = lane; i < nr; i += 32) acc += a[i] * xs[i];
        acc = warp_sum(acc);
        if (lane == 0) atomicAdd(&out[c], acc);
    }
}







// ---- eigen-decomposition of the symmetric tridiagonal T' (n <= kMaxKs) in one CTA of 512
// threads, all stages parallel over the eigenvalues:
//   1. eigenvalue i by multisection (8 threads, 9 sub-intervals per round, 19 rounds from the
//      Gershgorin interval: 9^-19 ~ 2^-60 of it) on the Sturm count of T' - x I;
//   2. its eigenvector by a twisted factorisation: pivots of the top-down and bottom-up LDL^T
//      of T' - lambda I, twist index r = argmin |gamma_r|, x_r = 1 and the two one-sided
//      recurrences (accurate for isolated eigenvalues);
//   3. classical Gram-Schmidt, twice, inside clusters (gaps < ctol ||T'||_1, default 1e-9,
//      LOVE_EIG_CTOL) for orthogonality;
//   4. W = V diag(sqrt(max(lambda, 0))) V^T.
// LOVE_JACOBI=1 switches to the cyclic Jacobi kernel below (4.4x slower at k' = 100, kept as a
// cross-check: tests/test_gpu_sampling.py compares the two roots).
// 1 / x to fp64 accuracy without the division subroutine: MUFU reciprocal + two Newton steps
// (|x| >= 1e-290 here: the pivots are floored at pivmin)
__device__ __forceinline__ double rcp64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(fma(-x, r, 1.0), r, r);
    r = fma(fma(-x, r, 1.0), r, r);
    return r;
}

// number of eigenvalues of T' below x: sign changes of the continuants
// p_k = (a_k - x) p_{k-1} - b_{k-1}^2 p_{k-2} (p_{-1} = 1), i.e. the negative pivots of the
// LDL^T of T' - x I, without divisions (rescaled every 8 terms); a zero counts as negative
__device__ __forceinline__ int sturm_count(const double* a, const double* b2, int n, double x) {
    double pm = 1.0, pc = a[0] - x;
    if (pc == 0.0) pc = -1e-300;                 // a zero pivot is taken as -tiny (negative)
    int cnt = pc < 0.0;
    // blocks of 8 terms (k = 8, 16, ... end a block: the rescale points), fully unrolled so the
    // shared-memory loads of a block issue ahead of the dependent chain
    for (int kb = 1; kb < n; kb += 8) {
        double ak[8], bk[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            ak[u] = kb + u < n ? a[kb + u] : 0.0;
            bk[u] = kb + u < n ? b2[kb + u - 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (kb + u < n) {
                double pn = (ak[u] - x) * pc - bk[u] * pm;
                if (pn == 0.0) pn = -1e-300 * pc;        // pivot p_k / p_{k-1} = -tiny
                cnt += (pn > 0.0) != (pc > 0.0);
                pm = pc;
                pc = pn;
            }
        }
        if (kb + 7 < n) {                         // k = kb + 7 = 8, 16, ...
            const double sc = rcp64(fabs(pc) + fabs(pm));
            pc *= sc;
            pm *= sc;
        }
    }
    return cnt;
}

// Gershgorin interval of T' (padded by 2 ulp), ||T'||_1 and max b_i^2 (thread 0)
__device__ __forceinline__ void gershgorin(const double* a, const double* b, const double* b2, int n, double* lo_out,
                                           double* hi_out, double* norm1, double* b2max) {
    double lo = 1e300, hi = -1e300, nrm = 0.0, bm = 0.0;
    for (int i = 0; i < n; ++i) {
        const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + fabs(b[i]);
        lo = fmin(lo, a[i] - r);
        hi = fmax(hi, a[i] + r);
        nrm = fmax(nrm, fabs(a[i]) + r);
        bm = fmax(bm, b2[i]);
    }
    const double pad = 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300;
    *lo_out = lo - pad;
    *hi_out = hi + pad;
    *norm1 = nrm;
    *b2max = bm;
}

// eigenvalue i of T' by multisection: the 8 lanes `sub` of an aligned lane group split the
// interval into 9 per round, 19 rounds from the Gershgorin interval (9^-19 ~ 2^-60 of it)
__device__ __forceinline__ double multisection(const double* a, const double* b2, int n, int i, int sub, double lo,
                                               double hi) {
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < 19; ++it) {
        const double x = lo + (hi - lo) * (double)(sub + 1) * (1.0 / 9.0);
        const int cnt = i < n ? sturm_count(a, b2, n, x) : 0;
        // new interval: between the last x with cnt <= i and the first x with cnt > i
        double nlo = lo, nhi = hi;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const double xt = __shfl_sync(0xffffffffu, x, (lane & ~7) + t);
            const int ct = __shfl_sync(0xffffffffu, cnt, (lane & ~7) + t);
            if (ct <= i) nlo = fmax(nlo, xt);
            else nhi = fmin(nhi, xt);
        }
        lo = nlo;
        hi = nhi;
    }
    return 0.5 * (lo + hi);
}

// Stage 1 spread over ceil(n / 8) CTAs (8 eigenvalues x 8 lanes each): the Sturm-count chains
// are FP64-pipe bound on one SM
__global__ void __launch_bounds__(64) tridiag_eigvals_kernel(const double* __restrict__ alpha,
                                                             const double* __restrict__ beta, int n,
                                                             double* __restrict__ lam) {
    __shared__ double a[kMaxKs], b[kMaxKs], b2[kMaxKs];
    __shared__ double s_lo, s_hi, s_norm1, s_b2max;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        a[i] = alpha[i];
        b[i] = i + 1 < n ? beta[i] : 0.0;
        b2[i] = b[i] * b[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) gershgorin(a, b, b2, n, &s_lo, &s_hi, &s_norm1, &s_b2max);
    __syncthreads();
    const int i = blockIdx.x * 8 + (threadIdx.x >> 3), sub = threadIdx.x & 7;
    const double l = multisection(a, b2, n, i, sub, s_lo, s_hi);
    if (i < n && sub == 0) lam[i] = l;
}

// lam_in != nullptr: the eigenvalues come from tridiag_eigvals_kernel (stage 1 skipped)
__global__ void __launch_bounds__(512) tridiag_root_kernel(const double* __restrict__ alpha,
                                                           const double* __restrict__ beta, int n,
                                                           double* __restrict__ Wout, double* __restrict__ evals,
                                                           double ctol, const double* __restrict__ lam_in) {
    __shared__ double a[kMaxKs], b[kMaxKs], b2[kMaxKs], lam[kMaxKs], sl[kMaxKs];
    extern __shared__ double Vsm[];                      // [n][n + 1], column i = eigenvector i
    const int LV = n + 1 + (n & 1 ? 1 : 0);     // odd: column sweeps spread over the banks
    __shared__ double s_lo, s_hi, s_norm1, s_b2max;
    __shared__ int cstart[kMaxKs];
    const int tid = threadIdx.x;
    for (int i = tid; i < n; i += blockDim.x) {
        a[i] = alpha[i];
        b[i] = i + 1 < n ? beta[i] : 0.0;
        b2[i] = b[i] * b[i];
        if (lam_in != nullptr) lam[i] = lam_in[i];
    }
    __syncthreads();
    if (tid == 0) gershgorin(a, b, b2, n, &s_lo, &s_hi, &s_norm1, &s_b2max);
    __syncthreads();
    const double pivmin = 1e-290 * fmax(1.0, s_b2max);
    // 1. multisection: 8 threads (sub) per eigenvalue i = tid / 8
    if (lam_in == nullptr) {
        for (int i0 = 0; i0 < n; i0 += 64) {
            const int i = i0 + (tid >> 3), sub = tid & 7;
            const double l = multisection(a, b2, n, i, sub, s_lo, s_hi);
            if (i < n && sub == 0) lam[i] = l;
        }
    }
    __syncthreads();
    // 2. twisted factorisation per eigenvalue (thread i)
    if (tid < n) {
        const int i = tid;
        const double l = lam[i];
        double dp[kMaxKs], dm[kMaxKs];
        dp[0] = a[0] - l;
        if (fabs(dp[0]) < pivmin) dp[0] = pivmin;
        for (int k = 1; k < n; ++k) {
            double d = (a[k] - l) - b2[k - 1] * rcp64(dp[k - 1]);
            if (fabs(d) < pivmin) d = pivmin;
            dp[k] = d;
        }
        dm[n - 1] = a[n - 1] - l;
        if (fabs(dm[n - 1]) < pivmin) dm[n - 1] = pivmin;
        for (int k = n - 2; k >= 0; --k) {
            double d = (a[k] - l) - b2[k] * rcp64(dm[k + 1]);
            if (fabs(d) < pivmin) d = pivmin;
            dm[k] = d;
        }
        int r = 0;
        double gmin = 1e300;
        for (int k = 0; k < n; ++k) {
            const double g = fabs(dp[k] + dm[k] - (a[k] - l));
            if (g < gmin) {
                gmin = g;
                r = k;
            }
        }
        double x = 1.0, nrm = 1.0;
        Vsm[(r) * LV + (i)] = 1.0;
        for (int k = r - 1; k >= 0; --k) {          // dp_k x_k + b_k x_{k+1} = 0
            x = -b[k] * x * rcp64(dp[k]);
            Vsm[(k) * LV + (i)] = x;
            nrm += x * x;
        }
        x = 1.0;
        for (int k = r + 1; k < n; ++k) {           // b_{k-1} x_{k-1} + dm_k x_k = 0
            x = -b[k - 1] * x * rcp64(dm[k]);
            Vsm[(k) * LV + (i)] = x;
            nrm += x * x;
        }
        const double inv = 1.0 / sqrt(nrm);
        for (int k = 0; k < n; ++k) Vsm[(k) * LV + (i)] *= inv;
    }
    __syncthreads();
    // 3. clusters (consecutive eigenvalues closer than ctol ||T'||_1): CGS twice per vector.
    // Twisted-factorisation vectors of eigenvalues a gap g apart are orthogonal to ~eps ||T'|| / g,
    // so ctol = 1e-9 leaves <= ~1e-7 non-orthogonality outside clusters
    if (tid == 0) {
        const double tol = ctol * s_norm1;
        int c0 = 0;
        for (int i = 0; i < n; ++i) {
            if (i > 0 && lam[i] - lam[i - 1] >= tol) c0 = i;
            cstart[i] = c0;
        }
    }
    __syncthreads();
    // one warp per cluster (clusters are independent): classical Gram-Schmidt, twice, of each
    // member against the earlier members, lanes over the n components
    const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    {
        int cl = 0;                                  // cluster ordinal of this warp's work
        for (int c0 = 0; c0 < n;) {
            int c1 = c0 + 1;
            while (c1 < n && cstart[c1] == c0) ++c1;
            if (c1 - c0 > 1 && (cl % nw) == wid) {
                for (int i = c0 + 1; i < c1; ++i)
                    for (int pass = 0; pass < 2; ++pass) {
                        for (int jj = c0; jj < i; ++jj) {
                            double d = 0.0;
                            for (int k = lane; k < n; k += 32) d += Vsm[k * LV + jj] * Vsm[k * LV + i];
                            d = warp_sum(d);
                            for (int k = lane; k < n; k += 32) Vsm[k * LV + i] -= d * Vsm[k * LV + jj];
                        }
                        double nn = 0.0;
                        for (int k = lane; k < n; k += 32) nn += Vsm[k * LV + i] * Vsm[k * LV + i];
                        nn = warp_sum(nn);
                        const double inv = 1.0 / sqrt(nn);
                        for (int k = lane; k < n; k += 32) Vsm[k * LV + i] *= inv;
                        __syncwarp();
                    }
            }
            if (c1 - c0 > 1) ++cl;
            c0 = c1;
        }
    }
    __syncthreads();
    // 4. W = V diag(sqrt(max(lambda, 0))) V^T
    for (int i = tid; i < n; i += blockDim.x) {
        evals[i] = lam[i];
        sl[i] = sqrt(fmax(lam[i], 0.0));
    }
    __syncthreads();
    double* U = Vsm + (size_t)n * LV;                    // U = V diag(sqrt(max(lambda, 0)))^(1/2)...
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int r = e / n, i = e - r * n;
        U[r * LV + i] = Vsm[r * LV + i] * sqrt(sl[i]);
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += blockDim.x) {      // W = U U^T = V diag(sqrt(lambda)) V^T
        const int r = e / n, c = e - r * n;
        const double* ur = U + r * LV;
        const double* uc = U + c * LV;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += ur[i] * uc[i];
        Wout[e] = acc;
    }
}

// ---- cyclic Jacobi eigensolver of the symmetric tridiagonal T' (n <= kMaxKs), one CTA.
// Parallel round-robin ordering: in each round the n/2 disjoint pairs (p, q) are rotated
// at once.  Output: W = V diag(sqrt(max(lambda, 0))) V^T (n x n, row-major) and lambda.
__global__ void __launch_bounds__(512) jacobi_root_kernel(const double* __restrict__ alpha,
                                                          const double* __restrict__ beta, int n,
                                                          double* __restrict__ Wout, double* __restrict__ evals) {
    extern __shared__ double sm[];
    const int N = n + (n & 1);                   // even order (a padded zero row/column)
    const int L = N + 1;                         // row stride: odd, so column sweeps hit distinct banks
    double* A = sm;                              // [N][L]
    double* V = A + N * L;                       // [N][L]
    double* cs = V + N * L;                      // [N/2] cos
    double* sn = cs + N / 2;                     // [N/2] sin
    int* pp = (int*)(sn + N / 2);                // [N/2]
    int* qq = pp + N / 2;                        // [N/2]
    __shared__ double offn;
    for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
        const int r = e / N, c = e % N;
        double v = 0.0;
        if (r < n && c < n) {
            if (r == c) v = alpha[r];
            else if (r == c + 1) v = beta[c];
            else if (c == r + 1) v = beta[r];
        }
        A[r * L + c] = v;
        V[r * L + c] = r == c ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int sweep = 0; sweep < 16; ++sweep) {
        if (threadIdx.x == 0) offn = 0.0;
        __syncthreads();
        double loc = 0.0, dia = 0.0;
        for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
            const int r = e / N, c = e % N;
            const double x = A[r * L + c];
            if (r != c) loc += x * x;
            else dia += x * x;
        }
        loc = warp_sum(loc);
        dia = warp_sum(dia);
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&offn, loc);
        }
        __syncthreads();
        __shared__ double diag_norm;
        if (threadIdx.x == 0) diag_norm = 0.0;
        __syncthreads();
        if ((threadIdx.x & 31) == 0) atomicAdd(&diag_norm, dia);
        __syncthreads();
        // converged: off-diagonal Frobenius norm <= 1e-11 of the diagonal's (eigenvalue errors
        // are quadratic in it; T' has a cluster of ~0 eigenvalues at breakdown that
        // keeps a tighter test from ever triggering -- measured: all 30 sweeps at 1e-13)
        if (offn <= 1e-22 * (diag_norm + 1e-300)) break;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
        for (int round = 0; round < N - 1; ++round) {
            // round-robin pairs: position 0 fixed, the others rotate
            for (int pi = threadIdx.x; pi < N / 2; pi += blockDim.x) {
                int a = pi == 0 ? 0 : 1 + (pi - 1 + round) % (N - 1);
                int b = 1 + (N - 2 - pi + round) % (N - 1);
                if (a > b) { const int t = a; a = b; b = t; }
                pp[pi] = a;
                qq[pi] = b;
                const double apq = A[a * L + b];
                double c = 1.0, s = 0.0;
                if (apq != 0.0) {
                    // t = tan of the rotation = sgn(theta) / (|theta| + sqrt(theta^2 + 1)),
                    // theta = d / (2 apq), d = a_bb - a_aa; written with one sqrt and one division
                    const double d = A[b * L + b] - A[a * L + a];
                    const double sg = (d == 0.0 || ((d > 0.0) == (apq > 0.0))) ? 1.0 : -1.0;
                    const double t = sg * 2.0 * fabs(apq) / (fabs(d) + sqrt(d * d + 4.0 * apq * apq));
                    c = rsqrt(t * t + 1.0);
                    s = t * c;
                }
                cs[pi] = c;
                sn[pi] = s;
            }
            __syncthreads();
            // rows: A <- J^T A (a warp per pair, lanes along the row)
            for (int pi = warp; pi < N / 2; pi += nwarp) {
                const int a = pp[pi], b = qq[pi];
                const double c = cs[pi], s = sn[pi];
                for (int col = lane; col < N; col += 32) {
                    const double xa = A[a * L + col], xb = A[b * L + col];
                    A[a * L + col] = c * xa - s * xb;
                    A[b * L + col] = s * xa + c * xb;
                }
            }
            __syncthreads();
            // columns: A <- A J, V <- V J (lanes down the column; the odd stride L spreads banks)
            for (int pi = warp; pi < N / 2; pi += nwarp) {
                const int a = pp[pi], b = qq[pi];
                const double c = cs[pi], s = sn[pi];
                for (int row = lane; row < N; row += 32) {
                    const double xa = A[row * L + a], xb = A[row * L + b];
                    A[row * L + a] = c * xa - s * xb;
                    A[row * L + b] = s * xa + c * xb;
                    const double va = V[row * L + a], vb = V[row * L + b];
                    V[row * L + a] = c * va - s * vb;
                    V[row * L + b] = s * va + c * vb;
                }
            }
            __syncthreads();
        }
    }
    double* sl = cs;                             // sqrt(max(lambda, 0)) (cs, sn are free now)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        evals[i] = A[i * L + i];
        sl[i] = sqrt(fmax(A[i * L + i], 0.0));
    }
    __syncthreads();
    // W[r][c] = sum_i V[r][i] sqrt(max(lambda_i, 0)) V[c][i]
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int r = e / n, c = e % n;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += V[r * L + i] * sl[i] * V[c * L + i];
        Wout[e] = acc;
    }
}

// S[row][c] = sum_i Q'[row + i*ldq] W[i][c]  -> V (fp32 / fp64) row-major m x ks_pad
// S = Q'~ diag(qscale) W (reading A18: S = Q' T'^{1/2}), 32 rows per CTA: the rows' Q' values
// (transposed, [i][row]) and W staged in shared memory; thread = (column c and c + 64, 8 rows),
// the 8 row values of each i read as one broadcast; the sum over i runs in ascending order as
// an FMA chain per output
constexpr int kRootRows = 32;
template <typename V>
__global__ void __launch_bounds__(256) root_tile_kernel(const double* __restrict__ Qp, int64_t ldq, int m, int n,
                                                        const double* __restrict__ qscale,
                                                        const double* __restrict__ W, int ks_pad, V* __restrict__ S) {
    extern __shared__ __align__(16) double sm[];
    double* Qt = sm;                              // [n][kRootRows]
    double* Ws = sm + (size_t)n * kRootRows;      // [n][ks_pad], columns >= n zero
    const int r0 = blockIdx.x * kRootRows;
    for (int e = threadIdx.x; e < n * ks_pad; e += blockDim.x) {
        const int i = e / ks_pad, c = e - i * ks_pad;
        Ws[e] = c < n ? W[i * n + c] : 0.0;
    }
    for (int e = threadIdx.x; e < kRootRows * n; e += blockDim.x) {
        const int i = e / kRootRows, r = e - i * kRootRows;     // coalesced along the rows of column i
        const int row = r0 + r;
        Qt[e] = row < m ? qscale[i] * Qp[(int64_t)i * ldq + row] : 0.0;
    }
    __syncthreads();
    const int c = threadIdx.x & 63, rg = threadIdx.x >> 6;    // rows rg*8 .. rg*8+7
    const bool c0 = c < ks_pad, c1 = c + 64 < ks_pad;
    double a0[8], a1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a0[u] = a1[u] = 0.0;
    for (int i = 0; i < n; ++i) {
        const double2* q2 = reinterpret_cast<const double2*>(Qt + i * kRootRows + rg * 8);
        double q[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double2 t = q2[u];
            q[2 * u] = t.x;
            q[2 * u + 1] = t.y;
        }
        const double w0 = c0 ? Ws[i * ks_pad + c] : 0.0;
        const double w1 = c1 ? Ws[i * ks_pad + c + 64] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0[u] = fma(q[u], w0, a0[u]);
            a1[u] = fma(q[u], w1, a1[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int row = r0 + rg * 8 + u;
        if (row >= m) break;
        if (c0) S[(int64_t)row * ks_pad + c] = (V)a0[u];
        if (c1) S[(int64_t)row * ks_pad + c + 64] = (V)a1[u];
    }
}

// ---- sampling-cache Lanczos on M v = K_UU v - Rc (Rc^T v) (Eqs. 12-13), run by the
// grid Lanczos machinery (device step index, CUDA-graph replay, the same reorthogonalisation
// kernels in fp64, two CGS passes); only the operator differs.  Q~ columns are unnormalised,
// q_j = qscale[j] Q~[:, j].

// v = z - Rc t (t = Rc^T q_j) and alpha_j += q_j . v   (fp64).  A CTA owns 32 rows; its 8
// warps split the k_eff columns (lanes over the rows: coalesced column reads), the partial sums
// meet in shared memory.  (One thread per row looping over every column left the kernel on 40
// SMs with a 49-load chain per thread.)
constexpr int kSvRows = 32;
__global__ void __launch_bounds__(256) samp_v_kernel(const double* __restrict__ Rc, int m, int k_eff,
                                                     const double* __restrict__ z, const double* __restrict__ t,
                                                     const double* __restrict__ qcur, double* __restrict__ v,
                                                     LanczosState st, double* __restrict__ t_next) {
    __shared__ double psum[8][kSvRows];
    pdl_wait();
    LOVE_TRACE(kTrSampV, *st.jdev);
    if (st.flags[0]) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r = blockIdx.x * kSvRows + lane;
    double acc = 0.0;
    if (r < m) {
        for (int c = wid; c < k_eff; c += 8) acc += Rc[(int64_t)c * m + r] * __ldg(&t[c]);
    }
    psum[wid][lane] = acc;
    __syncthreads();
    double a = 0.0;
    if (wid == 0 && r < m) {
        double tot = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) tot += psum[w][lane];
        const double vr = z[r] - tot;
        v[r] = vr;
        a = qcur[r] * vr;
    }
    if (wid == 0) {
        a = warp_sum(a);
        if (lane == 0) atomicAdd(st.alpha_cur, a);
    }
    // the other t buffer (read by the previous step, accumulated by the next) starts from zero
    if (blockIdx.x == 0)
        for (int c = threadIdx.x; c < k_eff; c += blockDim.x) t_next[c] = 0.0;
}

// q_j = s_j Q~'[:, j] (fp64) and t += Rc^T q_j over this CTA's kDotRows rows (dots_kernel's
// column loop; t was zeroed by the step before)
constexpr int kQdMaxRows = 256;
__global__ void __launch_bounds__(256) samp_qcur_dots_kernel(LanczosState st, const double* __restrict__ Q, int64_t ld,
                                                             int m, const double* __restrict__ Rc, int ncol,
                                                             double* __restrict__ qcur, double* __restrict__ t,
                                                             int rows) {
    pdl_wait();
    LOVE_TRACE(kTrMoments, *st.jdev);
    if (st.flags[0]) return;
    __shared__ double xs[kQdMaxRows];
    const int j = *st.jdev;
    const double sc = st.qscale[j];
    const int r0 = blockIdx.x * rows;
    const int nr = min(rows, m - r0);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
        const double q = sc * Q[(int64_t)j * ld + r0 + i];
        qcur[r0 + i] = q;
        xs[i] = q;
    }
    __syncthreads();
    // four columns per warp at a time: their loads and their warp reductions are independent
    // chains (one column at a time left a load -> shuffle-reduce -> atomic chain per column)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c0 = wid; c0 < ncol; c0 += 4 * nw) {
        double acc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + u * nw;
            acc[u] = 0.0;
            if (c < ncol) {
                const double* a = Rc + (int64_t)c * m + r0;
                for (int i = lane; i < nr; i += 32) acc[u] += a[i] * xs[i];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = warp_sum(acc[u]);
        if (lane == 0)
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c0 + u * nw < ncol) atomicAdd(&t[c0 + u * nw], acc[u]);
    }
}

__global__ void fill_ones_kernel(double* __restrict__ v, int m) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) v[i] = 1.0;
}

// ---- draws
struct Stencil1 {
    int base;
    double w[3][4];
    bool ok;
};

template <int D>
__device__ __forceinline__ Stencil1 stencil_at(const GridDev& g, const double* x) {
    Stencil1 s;
    s.ok = true;
    s.base = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int e = 0; e < 4; ++e) s.w[d][e] = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const double sc = (x[d] - g.lo[d]) / g.h[d];
        const double jf = floor(sc);
        const bool bad = !(jf >= 1.0 && jf <= (double)(g.m[d] - 3));
        s.ok = s.ok && !bad;
        const int j = bad ? 1 : (int)jf;
        keys4<double>(bad ? 0.0 : sc - jf, s.w[d]);
        s.base += (j - 1) * g.stride[d];
    }
    return s;
}

// G[i][c] = sum_l w_l S[node_l][c] (fp64 accumulation), mu[i] = sum_l w_l a[node_l]; warp per point
template <typename V, int D>
__global__ void __launch_bounds__(256) sample_gather_kernel(GridDev g, const V* __restrict__ S, int ks_pad, int ks,
                                                            const double* __restrict__ amean,
                                                            const double* __restrict__ Xs, int64_t t,
                                                            float* __restrict__ G, float* __restrict__ mu,
                                                            unsigned long long* __restrict__ counters) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= t) return;
    const Stencil1 st = stencil_at<D>(g, Xs + i * D);
    for (int c = lane; c < ks_pad; c += 32) {
        double acc = 0.0;
        if (st.ok && c < ks) {
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < (D > 1 ? 4 : 1); ++b)
                    for (int cc = 0; cc < (D > 2 ? 4 : 1); ++cc) {
                        int node = st.base + a * (D == 1 ? 1 : g.stride[0]);
                        double w = st.w[0][a];
                        if (D >= 2) { node += b * (D == 2 ? 1 : g.stride[1]); w *= st.w[1][b]; }
                        if (D == 3) { node += cc; w *= st.w[2][cc]; }
                        acc += w * (double)S[(int64_t)node * ks_pad + c];
                    }
        }
        G[i * ks_pad + c] = st.ok ? (float)acc : NAN;
    }
    if (lane == 0) {
        double m0 = 0.0;
        if (st.ok) {
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < (D > 1 ? 4 : 1); ++b)
                    for (int cc = 0; cc < (D > 2 ? 4 : 1); ++cc) {
                        int node = st.base + a * (D == 1 ? 1 : g.stride[0]);
                        double w = st.w[0][a];
                        if (D >= 2) { node += b * (D == 2 ? 1 : g.stride[1]); w *= st.w[1][b]; }
                        if (D == 3) { node += cc; w *= st.w[2][cc]; }
                        m0 += w * amean[node];
                    }
        } else {
            atomicAdd(&counters[1], 1ull);
        }
        mu[i] = st.ok ? (float)m0 : NAN;
    }
}

// Philox4x32-10 (counter-based, reading A24) and Box-Muller: zeta[c + j*ks_pad] ~ N(0, 1)
__device__ __forceinline__ uint4 philox4x32(uint4 ctr, uint2 key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned lo0 = 0xD2511F53u * ctr.x, hi0 = __umulhi(0xD2511F53u, ctr.x);
        const unsigned lo1 = 0xCD9E8D57u * ctr.z, hi1 = __umulhi(0xCD9E8D57u, ctr.z);
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
        key.x += 0x9E3779B9u;
        key.y += 0xBB67AE85u;
    }
    return ctr;
}

__global__ void philox_normal_kernel(uint64_t seed, int ks, int ks_pad, int64_t s, float* __restrict__ zeta) {
    // element e = j*ks + c (sample j, row c); 4 normals per Philox call
    const int64_t total = s * ks;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q * 4 < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = philox4x32(make_uint4((unsigned)q, (unsigned)(q >> 32), 0u, 0u),
                                   make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
        const unsigned u[4] = {r.x, r.y, r.z, r.w};
        float z[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float u1 = ((float)u[2 * h] + 1.0f) * 2.3283064365386963e-10f;   // (0, 1]
            const float u2 = (float)u[2 * h + 1] * 2.3283064365386963e-10f;
            const float rad = sqrtf(-2.0f * logf(u1));
            float sn, cs;
            sincospif(2.0f * u2, &sn, &cs);
            z[2 * h] = rad * cs;
            z[2 * h + 1] = rad * sn;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int64_t el = q * 4 + e;
            if (el < total) {
                const int64_t j = el / ks, c = el % ks;
                zeta[j * ks_pad + c] = z[e];
            }
        }
    }
}

__global__ void zeta_convert_kernel(const double* __restrict__ in, int ks, int ks_pad, int64_t s,
                                    float* __restrict__ zeta) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < s * ks_pad;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / ks_pad, c = e % ks_pad;
        zeta[e] = c < ks ? (float)in[j * ks + c] : 0.0f;
    }
}

// F[i + j*t] = mu[i] + sum_c G[i*ks_pad + c] zeta[j*ks_pad + c], register-blocked: CTA tile
// 128 points x 128 samples, 256 threads of 8 x 8 (two runs of 4 consecutive points x two runs
// of 4 samples, read from shared memory as 16-byte vectors), FFMA2 pairs along the points with
// the sample value broadcast; threads run along the points, so a warp's stores of one sample
// column are 256 contiguous bytes.
constexpr int kSgT = 128, kSgS = 128, kSgK = 16;

template <typename V>
__global__ void __launch_bounds__(256) sample_gemm2_kernel(const float* __restrict__ G, const float* __restrict__ Z,
                                                           const float* __restrict__ mu, int ks_pad, int64_t t,
                                                           int64_t s, V* __restrict__ F) {
    __shared__ __align__(16) float Gs[kSgK][kSgT + 4];
    __shared__ __align__(16) float Zs[kSgK][kSgS + 4];
    const int64_t i0 = (int64_t)blockIdx.x * kSgT, j0 = (int64_t)blockIdx.y * kSgS;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    f32x2 acc[4][8];                            // [point pair][sample]
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0ull;
    for (int k0 = 0; k0 < ks_pad; k0 += kSgK) {
        for (int e = threadIdx.x; e < kSgK * kSgT; e += 256) {
            const int r = e / kSgK, kk = e - r * kSgK;          // coalesced along k
            const int64_t gi = i0 + r, zj = j0 + r;
            Gs[kk][r] = (gi < t && k0 + kk < ks_pad) ? G[gi * ks_pad + k0 + kk] : 0.f;
            Zs[kk][r] = (zj < s && k0 + kk < ks_pad) ? Z[zj * ks_pad + k0 + kk] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kSgK; ++kk) {
            const float4 g0 = *reinterpret_cast<const float4*>(&Gs[kk][tx * 4]);
            const float4 g1 = *reinterpret_cast<const float4*>(&Gs[kk][64 + tx * 4]);
            const float4 z0 = *reinterpret_cast<const float4*>(&Zs[kk][ty * 4]);
            const float4 z1 = *reinterpret_cast<const float4*>(&Zs[kk][64 + ty * 4]);
            const f32x2 gp[4] = {pk2(g0.x, g0.y), pk2(g0.z, g0.w), pk2(g1.x, g1.y), pk2(g1.z, g1.w)};
            const float zv[8] = {z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w};
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const f32x2 zz = pk2(zv[b], zv[b]);
#pragma unroll
                for (int a = 0; a < 4; ++a) acc[a][b] = fma2(gp[a], zz, acc[a][b]);
            }
        }
        __syncthreads();
    }
    // rows: i0 + tx*4 + {0..3} (pairs 0, 1) and i0 + 64 + tx*4 + {0..3} (pairs 2, 3)
    float m4[8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int64_t gi = i0 + h * 64 + tx * 4 + e;
            m4[h * 4 + e] = gi < t ? mu[gi] : 0.f;
        }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const int64_t zj = j0 + (b < 4 ? ty * 4 + b : 64 + ty * 4 + (b - 4));
        if (zj >= s) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t gi = i0 + h * 64 + tx * 4;
            const float v0 = m4[h * 4 + 0] + lo2(acc[2 * h][b]), v1 = m4[h * 4 + 1] + hi2(acc[2 * h][b]);
            const float v2 = m4[h * 4 + 2] + lo2(acc[2 * h + 1][b]), v3 = m4[h * 4 + 3] + hi2(acc[2 * h + 1][b]);
            V* dst = F + zj * t + gi;
            if (std::is_same<V, float>::value && gi + 3 < t && ((zj * t + gi) & 3) == 0) {
                *reinterpret_cast<float4*>(dst) = make_float4(v0, v1, v2, v3);
            } else {
                if (gi < t) dst[0] = (V)v0;
                if (gi + 1 < t) dst[1] = (V)v1;
                if (gi + 2 < t) dst[2] = (V)v2;
                if (gi + 3 < t) dst[3] = (V)v3;
            }
        }
    }
}

}  // namespace

static __global__ void samp_flags_kernel(int* flags, int ks) {
    if (threadIdx.x == 0) {
        flags[0] = 0;
        flags[1] = ks;
        flags[2] = 0;
        flags[3] = 0;
    }
}

void build_sampling_cache(Cache& c, cudaStream_t s) {
    ProfScope ps(LOVE_PROF_SAMPLE_CACHE, s);
    const int ks = c.k_sample_req;
    const int m = c.g.m_total;
    const int k = c.k_eff;
    if (ks > kMaxKs) throw LoveError{LOVE_ERR_ARG, "k_sample must be <= 112"};
    const int64_t ldq = round_up(m, 2);
    const double* Rc = (const double*)c.Rc_col;      // m x k_eff, column-major (ld = m)
    double* Qp = (double*)dalloc(c, sizeof(double) * ldq * (ks + 1), s);
    double* v = (double*)dalloc(c, sizeof(double) * ldq, s);
    double* qcur = (double*)dalloc(c, sizeof(double) * (m + 4), s);
    double* z = (double*)dalloc(c, sizeof(double) * (m + 4), s);
    // t = Rc^T q_j, two buffers by step parity (a step accumulates one, its samp_v zeroes the other)
    double* tb[2];
    tb[0] = (double*)dalloc(c, sizeof(double) * 2 * std::max(k, 1), s);
    tb[1] = tb[0] + std::max(k, 1);
    // state of the M-Lanczos (reading A15: no Cholesky of T'; breakdown rule A12, tol 1e-10)
    LanczosState st{};
    {
        const size_t K = ks;
        double* p = (double*)dalloc(c, sizeof(double) * (1 + 1 + 2 * (K + 1) + 1 + (K + 1) + 5 * K + 2), s);
        st.alpha_cur = p; p += 1;
        st.beta2_cur = p; p += 1;
        st.c_cur = p; p += 2 * (K + 1);
        st.c_len = 2 * (int64_t)(K + 1);
        st.bnorm2 = p; p += 1;
        st.qscale = p; p += K + 1;
        st.alpha = p; p += K;
        st.beta = p; p += K;
        st.Ld = p; p += K;
        st.Ls = p; p += K;
        st.g = p; p += K;
        st.amax_bmax = p; p += 2;
        st.flags = (int*)dalloc(c, sizeof(int) * 8, s);
        st.jdev = st.flags + 4;
        st.step_ctr = st.flags + 5;
        st.chol = 0;
        if (std::getenv("LOVE_NO_DGKS") == nullptr) {   // DGKS-gated second CGS pass (lanczos.cu)
            st.nrm2 = (double*)dalloc(c, sizeof(double) * 2, s);
            st.dgks = std::getenv("LOVE_DGKS_LATE") ? 1 : 2;   // 2: the first pass decides (dgks_decide)
        }
        LOVE_LAUNCH(samp_flags_kernel, 1, 32, 0, s, st.flags, ks);
    }
    host_mark("samp_alloc");
    const double tol = 1e-10;
    const int gm = (int)ceil_div(m, kSvRows), gd = (int)ceil_div(m, kDotRows);
    const int gq = (int)std::min<int64_t>(ceil_div(m, 256), 148 * 4);
    // probe b' = M 1 (reading A14) into Q~[:, 0]
    LOVE_LAUNCH(fill_ones_kernel, gq, 256, 0, s, qcur, m);
    launch_kuu(c, qcur, z, s);
    LOVE_LAUNCH(dots_kernel, gd, 256, 0, s, Rc, (int64_t)m, m, k, qcur, tb[1], (const int*)nullptr);
    LOVE_LAUNCH(samp_v_kernel, gm, 256, 0, s, Rc, m, k, z, tb[1], qcur, Qp, st, tb[0]);
    LOVE_LAUNCH(dots_kernel, gd, 256, 0, s, Qp, ldq, m, 1, Qp, st.bnorm2, (const int*)nullptr);
    cuda_check(cudaMemsetAsync(st.alpha_cur, 0, sizeof(double), s), "alpha clear");
    launch_init_q0(st, s);
    // one step: q_j -> K_UU q_j, Rc^T q_j -> v, alpha -> two CGS passes (the last finalises)
    // rows per CTA of q_j / Rc^T q_j (fewer CTAs: fewer serialised fp64 atomics per column of
    // t; LOVE_QD_ROWS = 64 .. 256)
    const int qd_rows = std::getenv("LOVE_QD_ROWS") ? std::max(32, std::min(kQdMaxRows, std::atoi(std::getenv("LOVE_QD_ROWS"))))
                                                     : 128;
    int par = 0;
    auto step = [&]() {
        double* t = tb[par];
        LOVE_LAUNCH(samp_qcur_dots_kernel, (int)ceil_div(m, qd_rows), 256, 0, s, st, (const double*)Qp, ldq, m, Rc, k,
                    qcur, t, qd_rows);
        {
            DoneScope ds(st.flags);
            launch_kuu(c, qcur, z, s);
        }
        LOVE_LAUNCH(samp_v_kernel, gm, 256, 0, s, Rc, m, k, z, t, qcur, v, st, tb[par ^ 1]);
        par ^= 1;
        launch_reorth_pass_f64(st, Qp, ldq, m, ks, 0, 0, v, tol, s);
        launch_reorth_pass_f64(st, Qp, ldq, m, ks, 1, 1, v, tol, s);
    };
    const bool graph = !profiling() && std::getenv("LOVE_NO_GRAPH") == nullptr && ks >= 4;
    trace_begin(c, ks, s);
    ReplayThrottle thr(c.device);
    if (graph) st.hdone = thr.d;
    if (graph) {
        cudaGraph_t gph = nullptr;
        cudaGraphExec_t ge = nullptr;
        const int64_t before = g_launch_count.load();
        {   // every step kernel starts with pdl_wait(): programmatic dependent launch
            PdlScope pdl(std::getenv("LOVE_NO_PDL") == nullptr);
            cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "sampling capture");
            step();
            step();
            cuda_check(cudaStreamEndCapture(s, &gph), "sampling capture end");
        }
        host_mark("samp_capture");
        ge = graph_exec_cached(gph, "sampling/" + std::to_string(c.g.d) + "/" + std::to_string((int)st.dgks));
        host_mark("samp_instantiate");
        const int64_t nodes = g_launch_count.load() - before;
        g_launch_count -= nodes;
        // stop replaying after breakdown: the device sets the mapped host flag (ReplayThrottle),
        // a window of replays stays in flight, the stream is never drained to poll
        bool stop = false;
        for (int j = 0, i = 0; j + 1 < ks; j += 2, ++i) {
            if (!thr.admit(i)) {
                stop = true;
                break;
            }
            cuda_check(cudaGraphLaunch(ge, s), "sampling graph launch");
            g_launch_count += nodes;
            thr.launched(i, s);
        }
        if ((ks & 1) && !stop) step();
        cuda_check(cudaGraphDestroy(gph), "graph destroy");      // the exec stays cached
    } else {
        for (int j = 0; j < ks; ++j) step();
    }
    host_mark("samp_enqueued");
    if (c.trace != nullptr) trace_end(s);
    int hfl[4];
    cuda_check(cudaMemcpyAsync(hfl, st.flags, sizeof(hfl), cudaMemcpyDeviceToHost, s), "flags d2h");
    cuda_check(cudaStreamSynchronize(s), "sampling sync");
    host_mark("samp_sync");
    trace_report(c, hfl[0] ? hfl[1] : ks);
    if (hfl[3]) throw LoveError{LOVE_ERR_ZERO_PROBE, "sampling probe M 1 is zero"};
    // every step that ran to the end set done at i = ks - 1 or at the breakdown step
    const int ke = hfl[0] ? hfl[1] : ks;
    c.k_sample_eff = ke;
    c.ks_pad = (int)round_up(std::max(ke, 1), 4);
    double* W = (double*)dalloc(c, sizeof(double) * ke * ke, s);
    double* ev = (double*)dalloc(c, sizeof(double) * ke, s);
    const int N = ke + (ke & 1);
    const size_t smj = sizeof(double) * (2 * (size_t)N * (N + 1) + N) + sizeof(int) * N;
    if (std::getenv("LOVE_JACOBI") != nullptr) {
        ensure_smem((const void*)jacobi_root_kernel, smj);
        LOVE_LAUNCH(jacobi_root_kernel, 1, 512, smj, s, st.alpha, st.beta, ke, W, ev);
    } else {
        const size_t smv = sizeof(double) * 2 * (size_t)ke * (ke + 2);
        // the opt-in limit counts static + dynamic shared memory (the kernel's static arrays
        // are ~6 KB): request it whenever the sum passes 48 KB
        ensure_smem((const void*)tridiag_root_kernel, smv + 8192);
        static const bool one_cta = std::getenv("LOVE_EIG_ONE_CTA") != nullptr;
        if (!one_cta) LOVE_LAUNCH(tridiag_eigvals_kernel, (int)ceil_div(ke, 8), 64, 0, s, st.alpha, st.beta, ke, ev);
        LOVE_LAUNCH(tridiag_root_kernel, 1, 512, smv, s, st.alpha, st.beta, ke, W, ev,
                    std::getenv("LOVE_EIG_CTOL") ? std::atof(std::getenv("LOVE_EIG_CTOL")) : 1e-9,
                    one_cta ? (const double*)nullptr : (const double*)ev);
    }
    c.S = dalloc(c, c.vsize * (size_t)m * c.ks_pad, s);
    // S = Q' diag(qscale) W, 32 rows per CTA (the rows' Q' values and W staged in shared memory)
    const size_t smr = sizeof(double) * ((size_t)ke * c.ks_pad + (size_t)kRootRows * ke);
    const int gr = (int)ceil_div(m, kRootRows);
    if (c.precision == LOVE_FP64) {
        ensure_smem((const void*)root_tile_kernel<double>, smr);
        LOVE_LAUNCH(root_tile_kernel<double>, gr, 256, smr, s, Qp, ldq, m, ke, st.qscale, W, c.ks_pad, (double*)c.S);
    } else {
        ensure_smem((const void*)root_tile_kernel<float>, smr);
        LOVE_LAUNCH(root_tile_kernel<float>, gr, 256, smr, s, Qp, ldq, m, ke, st.qscale, W, c.ks_pad, (float*)c.S);
    }
    c.h_evals.resize(ke);
    cuda_check(cudaMemcpyAsync(c.h_evals.data(), ev, sizeof(double) * ke, cudaMemcpyDeviceToHost, s), "evals");
    cuda_check(cudaStreamSynchronize(s), "sampling sync");
    host_mark("samp_root");
}

template <typename VS>
void launch_sample_gather(const Cache& c, const double* Xs, int64_t t, float* G, float* mu, int gb, cudaStream_t s) {
    const int ks = c.k_sample_eff, kp = c.ks_pad;
    switch (c.g.d) {
        case 1: LOVE_LAUNCH((sample_gather_kernel<VS, 1>), gb, 256, 0, s, c.g, (const VS*)c.S, kp, ks,
                            (const double*)c.a, Xs, t, G, mu, c.counters); break;
        case 2: LOVE_LAUNCH((sample_gather_kernel<VS, 2>), gb, 256, 0, s, c.g, (const VS*)c.S, kp, ks,
                            (const double*)c.a, Xs, t, G, mu, c.counters); break;
        default: LOVE_LAUNCH((sample_gather_kernel<VS, 3>), gb, 256, 0, s, c.g, (const VS*)c.S, kp, ks,
                             (const double*)c.a, Xs, t, G, mu, c.counters); break;
    }
}

template <typename V>
void launch_sample(const Cache& c, const double* Xs, int64_t t, int64_t ns, uint64_t seed, const double* zeta,
                   V* out, cudaStream_t s) {
    if (t <= 0 || ns <= 0) return;
    ProfScope ps(LOVE_PROF_SAMPLE, s);
    const int ks = c.k_sample_eff, kp = c.ks_pad;
    float *G = nullptr, *mu = nullptr, *Z = nullptr;
    cuda_check(cudaMallocAsync((void**)&G, sizeof(float) * t * kp, s), "sample alloc");
    cuda_check(cudaMallocAsync((void**)&mu, sizeof(float) * t, s), "sample alloc");
    cuda_check(cudaMallocAsync((void**)&Z, sizeof(float) * ns * kp, s), "sample alloc");
    const int gb = (int)ceil_div(t * 32, 256);
    // S is stored in the cache precision (double for LOVE_FP64 and opts.cache_fp64 caches)
    if (c.precision == LOVE_FP64) launch_sample_gather<double>(c, Xs, t, G, mu, gb, s);
    else launch_sample_gather<float>(c, Xs, t, G, mu, gb, s);
    if (zeta) {
        LOVE_LAUNCH(zeta_convert_kernel, (int)std::min<int64_t>(ceil_div(ns * kp, 256), 4096), 256, 0, s, zeta, ks, kp,
                    ns, Z);
    } else {
        cuda_check(cudaMemsetAsync(Z, 0, sizeof(float) * ns * kp, s), "zeta zero");
        LOVE_LAUNCH(philox_normal_kernel, (int)std::min<int64_t>(ceil_div(ns * ks, 1024), 4096), 256, 0, s, seed, ks, kp,
                    ns, Z);
    }
    const dim3 grid((unsigned)ceil_div(t, kSgT), (unsigned)ceil_div(ns, kSgS));
    prof_begin(LOVE_PROF_SAMPLE_GEMM, s);
    LOVE_LAUNCH(sample_gemm2_kernel<V>, grid, 256, 0, s, G, Z, mu, kp, t, ns, out);
    prof_end(LOVE_PROF_SAMPLE_GEMM, s);
    cuda_check(cudaFreeAsync(G, s), "sample free");
    cuda_check(cudaFreeAsync(mu, s), "sample free");
    cuda_check(cudaFreeAsync(Z, s), "sample free");
}

template void launch_sample<float>(const Cache&, const double*, int64_t, int64_t, uint64_t, const double*, float*,
                                   cudaStream_t);
template void launch_sample<double>(const Cache&, const double*, int64_t, int64_t, uint64_t, const double*,
                                    double*, cudaStream_t);

}  // namespace love
