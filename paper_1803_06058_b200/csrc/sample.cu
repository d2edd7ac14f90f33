// sample.cu -- posterior sampling with LOVE (Eqs. 11-15).
//
// Sampling cache (build time, fp64, reading A16):
//   M v = K_UU v - Rc (Rc^T v)            (Eq. 12 / 13: K_UU - R^T R', Rc Rc^T = R^T R')
//   k' Lanczos steps on M from b' = M 1 (reading A14), three-term + CGS2,
//   breakdown rule of reading A12  ->  Q' (m x k'), T' (k' x k')
//   T' = V diag(lambda) V^T (cyclic Jacobi, one CTA), T'^{1/2} = V diag(sqrt(max(lambda, 0))) V^T
//   S = Q' T'^{1/2}  (reading A15: the unique PSD root replaces the Cholesky factor of P:351)
// Draws (love_sample):
//   G = W_{X*}^T S (t x k'),  mu = W_{X*}^T a,  F = mu 1^T + G zeta    (Eq. 11)
//   zeta from the caller (shared-draw parity) or Philox4x32-10 + Box-Muller (reading A24).
#include <cuda_runtime.h>

#include <cmath>

#include "love_internal.h"

namespace love {

namespace {

constexpr int kMaxKs = 112;          // k' limit of the single-CTA Jacobi eigensolver (smem)

// out[c] += sum_r A[r + c*lda] * x[r], c < ncol   (fp64, CTA row tiles, warps own columns)
constexpr int kDotRows = 128;       // rows per CTA tile of dots_kernel (~m/128 CTAs)
__global__ void __launch_bounds__(256) dots_kernel(const double* __restrict__ A, int64_t lda, int nrow, int ncol,
                                                   const double* __restrict__ x, double* __restrict__ out,
                                                   const int* __restrict__ stop) {
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

// out[r] = base[r] - sum_c A[r + c*lda] * coef[c] * cscale   (base may alias out)
__global__ void __launch_bounds__(256) sub_kernel(const double* base, const double* __restrict__ A, int64_t lda,
                                                  int nrow, int ncol, const double* __restrict__ coef, double* out,
                                                  const int* __restrict__ stop) {
    if (stop && *stop) return;
    extern __shared__ double cs[];               // [ncol]
    for (int i = threadIdx.x; i < ncol; i += blockDim.x) cs[i] = coef[i];
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrow) return;
    double acc = 0.0;
    for (int c = 0; c < ncol; ++c) acc += A[(int64_t)c * lda + r] * cs[c];
    out[r] = base[r] - acc;
}

// Lanczos scalars of the sampling cache (one thread), state layout:
//   st[0] alpha acc, st[1] beta2 acc (both per step slot), see SampState
struct SampState {
    double* alpha;      // [ks]
    double* beta;       // [ks]
    double* acc;        // [ks][4 + 2*(ks+1) + (k+1)] per-step accumulators
    int* flags;         // [4] done, k_eff, zero probe
    double* amax_bmax;  // [2]
};

__host__ __device__ inline int64_t samp_slot(int ks, int k) { return 4 + 2 * (ks + 1) + (k + 1); }

// v -= alpha_j q_j + beta_{j-1} q_{j-1}   (alpha_j = acc[0] of step j)
__global__ void three_term_kernel(double* __restrict__ v, const double* __restrict__ Qp, int64_t ldq, int m, int j,
                                  SampState s, int ks, int k) {
    if (s.flags[0]) return;
    const double* acc = s.acc + (int64_t)j * samp_slot(ks, k);
    const double al = acc[0];
    const double bt = j > 0 ? s.beta[j - 1] : 0.0;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r == 0 && blockIdx.x == 0) s.alpha[j] = al;
    if (r >= m) return;
    double x = v[r] - al * Qp[(int64_t)j * ldq + r];
    if (j > 0) x -= bt * Qp[(int64_t)(j - 1) * ldq + r];
    v[r] = x;
}

// beta_j = ||v||, breakdown test, q_{j+1} = v / beta_j
__global__ void normalize_kernel(const double* __restrict__ v, double* __restrict__ Qp, int64_t ldq, int m, int j,
                                 SampState s, int ks, int k, double tol) {
    if (s.flags[0]) return;
    const double* acc = s.acc + (int64_t)j * samp_slot(ks, k);
    const double b = sqrt(acc[1]);
    const double amax = fmax(s.amax_bmax[0], fabs(s.alpha[j]));
    const double bmax = fmax(s.amax_bmax[1], b);
    const bool stop = !(b >= tol * (amax + 2.0 * bmax));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s.amax_bmax[0] = amax;
        s.amax_bmax[1] = bmax;
    }
    __syncthreads();
    if (stop) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            s.flags[0] = 1;
            s.flags[1] = j + 1;
        }
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) s.beta[j] = b;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) Qp[(int64_t)(j + 1) * ldq + r] = v[r] / b;
}

__global__ void probe_init_kernel(double* __restrict__ v, int m) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) v[i] = 1.0;
}

__global__ void probe_normalize_kernel(const double* __restrict__ v, double* __restrict__ Qp, int m,
                                       const double* __restrict__ n2, SampState s) {
    const double nb = sqrt(*n2);
    if (!(nb > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            s.flags[0] = 1;
            s.flags[1] = 0;
            s.flags[2] = 1;
        }
        return;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) Qp[i] = v[i] / nb;
}

// ---- cyclic Jacobi eigensolver of the symmetric tridiagonal T' (n <= kMaxKs), one CTA.
// Parallel round-robin ordering: in each round the n/2 disjoint pairs (p, q) are rotated
// at once.  Output: W = V diag(sqrt(max(lambda, 0))) V^T (n x n, row-major) and lambda.
__global__ void __launch_bounds__(512) jacobi_root_kernel(const double* __restrict__ alpha,
                                                          const double* __restrict__ beta, int n,
                                                          double* __restrict__ Wout, double* __restrict__ evals) {
    extern __shared__ double sm[];
    const int N = n + (n & 1);                   // even order (a padded zero row/column)
    double* A = sm;                              // [N][N]
    double* V = A + N * N;                       // [N][N]
    double* cs = V + N * N;                      // [N/2] cos
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
        A[e] = v;
        V[e] = r == c ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int sweep = 0; sweep < 30; ++sweep) {
        if (threadIdx.x == 0) offn = 0.0;
        __syncthreads();
        double loc = 0.0, dia = 0.0;
        for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
            const int r = e / N, c = e % N;
            if (r != c) loc += A[e] * A[e];
            else dia += A[e] * A[e];
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
        // converged: off-diagonal Frobenius norm <= 1e-13 of the diagonal's (fp64 round-off of
        // the rotations is ~1e-15 per sweep; the root only needs T'^{1/2} to ~1e-12)
        if (offn <= 1e-26 * (diag_norm + 1e-300)) break;
        for (int round = 0; round < N - 1; ++round) {
            // round-robin pairs: position 0 fixed, the others rotate
            for (int pi = threadIdx.x; pi < N / 2; pi += blockDim.x) {
                int a = pi == 0 ? 0 : 1 + (pi - 1 + round) % (N - 1);
                int b = 1 + (N - 2 - pi + round) % (N - 1);
                if (a > b) { const int t = a; a = b; b = t; }
                pp[pi] = a;
                qq[pi] = b;
                const double apq = A[a * N + b];
                double c = 1.0, s = 0.0;
                if (apq != 0.0) {
                    const double theta = (A[b * N + b] - A[a * N + a]) / (2.0 * apq);
                    const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                    c = 1.0 / sqrt(t * t + 1.0);
                    s = t * c;
                }
                cs[pi] = c;
                sn[pi] = s;
            }
            __syncthreads();
            // rows: A <- J^T A
            for (int e = threadIdx.x; e < (N / 2) * N; e += blockDim.x) {
                const int pi = e / N, col = e % N;
                const int a = pp[pi], b = qq[pi];
                const double c = cs[pi], s = sn[pi];
                const double xa = A[a * N + col], xb = A[b * N + col];
                A[a * N + col] = c * xa - s * xb;
                A[b * N + col] = s * xa + c * xb;
            }
            __syncthreads();
            // columns: A <- A J, V <- V J
            for (int e = threadIdx.x; e < (N / 2) * N; e += blockDim.x) {
                const int pi = e / N, row = e % N;
                const int a = pp[pi], b = qq[pi];
                const double c = cs[pi], s = sn[pi];
                const double xa = A[row * N + a], xb = A[row * N + b];
                A[row * N + a] = c * xa - s * xb;
                A[row * N + b] = s * xa + c * xb;
                const double va = V[row * N + a], vb = V[row * N + b];
                V[row * N + a] = c * va - s * vb;
                V[row * N + b] = s * va + c * vb;
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) evals[i] = A[i * N + i];
    __syncthreads();
    // W[r][c] = sum_i V[r][i] sqrt(max(lambda_i, 0)) V[c][i]
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int r = e / n, c = e % n;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += V[r * N + i] * sqrt(fmax(A[i * N + i], 0.0)) * V[c * N + i];
        Wout[e] = acc;
    }
}

// S[row][c] = sum_i Q'[row + i*ldq] W[i][c]  -> V (fp32 / fp64) row-major m x ks_pad
template <typename V>
__global__ void __launch_bounds__(256) root_kernel(const double* __restrict__ Qp, int64_t ldq, int m, int n,
                                                   const double* __restrict__ W, int ks_pad, V* __restrict__ S) {
    extern __shared__ double Ws[];               // [n][n]
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Ws[e] = W[e];
    __syncthreads();
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= m) return;
    double q[kMaxKs];
    for (int i = 0; i < n; ++i) q[i] = Qp[(int64_t)i * ldq + row];
    for (int c = lane; c < ks_pad; c += 32) {
        double acc = 0.0;
        if (c < n)
            for (int i = 0; i < n; ++i) acc += q[i] * Ws[i * n + c];
        S[(int64_t)row * ks_pad + c] = (V)acc;
    }
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

// F[i + j*t] = mu[i] + sum_c G[i*ks_pad + c] zeta[j*ks_pad + c]    (FP32 FMA tiles, no tensor cores)
// CTA tile: 64 points x 64 samples, 256 threads each computing 4 x 4; K staged 16 at a time.
template <typename V>
__global__ void __launch_bounds__(256) sample_gemm_kernel(const float* __restrict__ G, const float* __restrict__ Z,
                                                          const float* __restrict__ mu, int ks_pad, int64_t t,
                                                          int64_t s, V* __restrict__ F) {
    __shared__ float Gs[16][64 + 4];
    __shared__ float Zs[16][64 + 4];
    const int64_t i0 = (int64_t)blockIdx.x * 64, j0 = (int64_t)blockIdx.y * 64;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;      // 16 x 16 threads
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < ks_pad; k0 += 16) {
        for (int e = threadIdx.x; e < 16 * 64; e += 256) {
            const int r = e / 16, kk = e % 16;                  // coalesced along k
            const int64_t gi = i0 + r, zj = j0 + r;
            Gs[kk][r] = (gi < t && k0 + kk < ks_pad) ? G[gi * ks_pad + k0 + kk] : 0.f;
            Zs[kk][r] = (zj < s && k0 + kk < ks_pad) ? Z[zj * ks_pad + k0 + kk] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float ga[4], zb[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) ga[a] = Gs[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) zb[b] = Zs[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] += ga[a] * zb[b];
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int64_t gi = i0 + ty + 16 * a;
        if (gi >= t) continue;
        const float m0 = mu[gi];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t zj = j0 + tx + 16 * b;
            if (zj < s) F[zj * t + gi] = (V)(m0 + acc[a][b]);
        }
    }
}

}  // namespace

void build_sampling_cache(Cache& c, cudaStream_t s) {
    ProfScope ps(LOVE_PROF_SAMPLE_CACHE, s);
    ensure_smem((const void*)sub_kernel, sizeof(double) * std::max(c.k_eff, c.k_sample_req + 1));
    const int ks = c.k_sample_req;
    const int m = c.g.m_total;
    const int k = c.k_eff;
    if (ks > kMaxKs) throw LoveError{LOVE_ERR_ARG, "k_sample must be <= 112"};
    const int64_t ldq = round_up(m, 2);
    const double* Rc = (const double*)c.Rc_col;      // m x k_eff, column-major (ld = m)
    double* Qp = (double*)dalloc(c, sizeof(double) * ldq * (ks + 1), s);
    double* v = (double*)dalloc(c, sizeof(double) * ldq, s);
    double* z = (double*)dalloc(c, sizeof(double) * (ldq + 4), s);
    SampState st;
    st.alpha = (double*)dalloc(c, sizeof(double) * ks, s);
    st.beta = (double*)dalloc(c, sizeof(double) * ks, s);
    const int64_t slot = samp_slot(ks, k);
    st.acc = (double*)dalloc(c, sizeof(double) * (ks + 1) * slot, s);
    st.flags = (int*)dalloc(c, sizeof(int) * 4, s);
    st.amax_bmax = (double*)dalloc(c, sizeof(double) * 2, s);
    {
        const int kk = ks;
        cuda_check(cudaMemcpyAsync(st.flags + 1, &kk, sizeof(int), cudaMemcpyHostToDevice, s), "flags");
    }
    const int gm = (int)ceil_div(m, 256), gd = (int)ceil_div(m, kDotRows);
    double* n2 = st.acc + (int64_t)ks * slot;          // spare slot: ||M 1||^2
    // M v for a vector x: z = K_UU x ; t = Rc^T x ; out = z - Rc t
    auto apply_M = [&](const double* x, double* out, double* tacc) {
        launch_kuu(c, x, z, s);
        LOVE_LAUNCH(dots_kernel, gd, 256, 0, s, Rc, (int64_t)m, m, k, x, tacc, st.flags);
        LOVE_LAUNCH(sub_kernel, gm, 256, sizeof(double) * k, s, z, Rc, (int64_t)m, m, k, tacc, out, st.flags);
    };
    // probe b' = M 1 (reading A14)
    LOVE_LAUNCH(probe_init_kernel, gm, 256, 0, s, v, m);
    apply_M(v, v, n2 + 4);
    LOVE_LAUNCH(dots_kernel, gd, 256, 0, s, v, (int64_t)ldq, m, 1, v, n2, (const int*)nullptr);
    LOVE_LAUNCH(probe_normalize_kernel, gm, 256, 0, s, v, Qp, m, n2, st);
    int* hflag = nullptr;                               // pinned: breakdown polled every 8 steps
    cuda_check(cudaMallocHost((void**)&hflag, sizeof(int)), "pinned flag");
    for (int j = 0; j < ks; ++j) {
        if (j > 0 && (j & 7) == 0) {   // stop issuing steps once the M-Lanczos has broken down (A12)
            cuda_check(cudaMemcpyAsync(hflag, st.flags, sizeof(int), cudaMemcpyDeviceToHost, s), "flag poll");
            cuda_check(cudaStreamSynchronize(s), "flag poll");
            if (*hflag) break;
        }
        double* acc = st.acc + (int64_t)j * slot;      // [0] alpha, [1] beta^2, [4..] CGS dots, then Rc^T q
        const double* qj = Qp + (int64_t)j * ldq;
        apply_M(qj, v, acc + 4 + 2 * (ks + 1));
        LOVE_LAUNCH(dots_kernel, gd, 256, 0, s, qj, (int64_t)ldq, m, 1, v, acc, st.flags);   // alpha_j
        LOVE_LAUNCH(three_term_kernel, gm, 256, 0, s, v, Qp, ldq, m, j, st, ks, k);
        if (j == ks - 1) {
            // alpha of the last step is recorded by three_term_kernel; no new vector
            break;
        }
        for (int pass = 0; pass < 2; ++pass) {                                        // CGS2
            double* cp = acc + 4 + pass * (ks + 1);
            LOVE_LAUNCH(dots_kernel, gd, 256, 0, s, Qp, ldq, m, j + 1, v, cp, st.flags);
            LOVE_LAUNCH(sub_kernel, gm, 256, sizeof(double) * (j + 1), s, v, Qp, ldq, m, j + 1, cp, v, st.flags);
        }
        LOVE_LAUNCH(dots_kernel, gd, 256, 0, s, v, (int64_t)ldq, m, 1, v, acc + 1, st.flags);   // beta^2
        LOVE_LAUNCH(normalize_kernel, gm, 256, 0, s, v, Qp, ldq, m, j, st, ks, k, 1e-10);
    }
    int hfl[4];
    cuda_check(cudaMemcpyAsync(hfl, st.flags, sizeof(hfl), cudaMemcpyDeviceToHost, s), "flags d2h");
    cuda_check(cudaStreamSynchronize(s), "sampling sync");
    cudaFreeHost(hflag);
    if (hfl[2]) throw LoveError{LOVE_ERR_ZERO_PROBE, "sampling probe M 1 is zero"};
    const int ke = hfl[0] ? hfl[1] : ks;
    c.k_sample_eff = ke;
    c.ks_pad = (int)round_up(std::max(ke, 1), 4);
    double* W = (double*)dalloc(c, sizeof(double) * ke * ke, s);
    double* ev = (double*)dalloc(c, sizeof(double) * ke, s);
    const int N = ke + (ke & 1);
    const size_t smj = sizeof(double) * (2 * (size_t)N * N + N) + sizeof(int) * N;
    ensure_smem((const void*)jacobi_root_kernel, smj);
    LOVE_LAUNCH(jacobi_root_kernel, 1, 512, smj, s, st.alpha, st.beta, ke, W, ev);
    c.S = dalloc(c, c.vsize * (size_t)m * c.ks_pad, s);
    const size_t smr = sizeof(double) * ke * ke;
    if (c.precision == LOVE_FP64) {
        ensure_smem((const void*)root_kernel<double>, smr);
        LOVE_LAUNCH(root_kernel<double>, (int)ceil_div(m, 8), 256, smr, s, Qp, ldq, m, ke, W, c.ks_pad, (double*)c.S);
    } else {
        ensure_smem((const void*)root_kernel<float>, smr);
        LOVE_LAUNCH(root_kernel<float>, (int)ceil_div(m, 8), 256, smr, s, Qp, ldq, m, ke, W, c.ks_pad, (float*)c.S);
    }
    c.h_evals.resize(ke);
    cuda_check(cudaMemcpyAsync(c.h_evals.data(), ev, sizeof(double) * ke, cudaMemcpyDeviceToHost, s), "evals");
    cuda_check(cudaStreamSynchronize(s), "sampling sync");
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
    switch (c.g.d) {
        case 1: LOVE_LAUNCH((sample_gather_kernel<V, 1>), gb, 256, 0, s, c.g, (const V*)c.S, kp, ks, (const double*)c.a,
                            Xs, t, G, mu, c.counters); break;
        case 2: LOVE_LAUNCH((sample_gather_kernel<V, 2>), gb, 256, 0, s, c.g, (const V*)c.S, kp, ks, (const double*)c.a,
                            Xs, t, G, mu, c.counters); break;
        default: LOVE_LAUNCH((sample_gather_kernel<V, 3>), gb, 256, 0, s, c.g, (const V*)c.S, kp, ks, (const double*)c.a,
                             Xs, t, G, mu, c.counters); break;
    }
    if (zeta) {
        LOVE_LAUNCH(zeta_convert_kernel, (int)std::min<int64_t>(ceil_div(ns * kp, 256), 4096), 256, 0, s, zeta, ks, kp,
                    ns, Z);
    } else {
        cuda_check(cudaMemsetAsync(Z, 0, sizeof(float) * ns * kp, s), "zeta zero");
        LOVE_LAUNCH(philox_normal_kernel, (int)std::min<int64_t>(ceil_div(ns * ks, 1024), 4096), 256, 0, s, seed, ks, kp,
                    ns, Z);
    }
    dim3 grid((unsigned)ceil_div(t, 64), (unsigned)ceil_div(ns, 64));
    LOVE_LAUNCH(sample_gemm_kernel<V>, grid, 256, 0, s, G, Z, mu, kp, t, ns, out);
    cuda_check(cudaFreeAsync(G, s), "sample free");
    cuda_check(cudaFreeAsync(mu, s), "sample free");
    cuda_check(cudaFreeAsync(Z, s), "sample free");
}

template void launch_sample<float>(const Cache&, const double*, int64_t, int64_t, uint64_t, const double*, float*,
                                   cudaStream_t);
template void launch_sample<double>(const Cache&, const double*, int64_t, int64_t, uint64_t, const double*,
                                    double*, cudaStream_t);

}  // namespace love
