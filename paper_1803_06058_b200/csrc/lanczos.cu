// lanczos.cu -- the Lanczos driver with full reorthogonalisation, the streamed Cholesky of
// T_k and the streamed LOVE cache Rc.
//
// Step j (0-based; q_j = qscale[j] * Q~[:, j], columns of Q~ are stored unnormalised):
//   scatter u = W q_j ; z_j = K_UU u ; r = W^T z_j + sigma^2 q_j ; alpha_j = q_j^T r
//   r' = r - alpha_j q_j - beta_{j-1} q_{j-1}                      (three-term)
//   c = Q_j^T r' ; q~_{j+1} = r' - Q_j c   (full reorthogonalisation; reading A10:
//                                            one pass in fp32, two in fp64 = CGS2)
//   beta_j = ||q~_{j+1}|| ; breakdown if beta_j < tol (max|alpha| + 2 max beta) (A12)
// Streamed cache (reading A9): with T_k = L L^T and z_j = K_UU W q_j (a free
// by-product of the MVM), Rc[:, j] = (z_j - L_{j,j-1} Rc[:, j-1]) / L_jj, so that
// Rc = K_UU W Q_k L^{-T} and Rc Rc^T = R^T R' of P:282-285.  Mean cache (Eq. 6 via Eq. 3,
// probe y): a = ||y|| Rc L^{-1} e_1, also streamed.
#include <cuda_runtime.h>
#include <cstdio>

#include <algorithm>
#include <cstdlib>
#include <memory>

#include "love_internal.h"

#ifndef LOVE_SWEEP_NB
#define LOVE_SWEEP_NB 1
#endif
#ifndef LOVE_UPD_B
#define LOVE_UPD_B 8
#endif
namespace love {

LOVE_TRACE_TU(lanczos)
constexpr int kUpdB = LOVE_UPD_B;
constexpr int kCondSteps = 2;
template <typename V> int update_grid(int64_t nchunks, size_t smem, int cg);
int update_groups(int64_t nchunks);
}

namespace love {

namespace {

template <typename V> struct VecT;
template <> struct VecT<float> { using T = float4; static constexpr int W = 4; };
template <> struct VecT<double> { using T = double2; static constexpr int W = 2; };

template <typename V>
__device__ __forceinline__ void vload(const V* p, V out[VecT<V>::W]) {
    using T = typename VecT<V>::T;
    const T v = *reinterpret_cast<const T*>(p);
    if constexpr (VecT<V>::W == 4) { out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w; }
    else { out[0] = v.x; out[1] = v.y; }
}

template <typename V>
__device__ __forceinline__ void vstore(V* p, const V in[VecT<V>::W]) {
    using T = typename VecT<V>::T;
    T v;
    if constexpr (VecT<V>::W == 4) { v.x = in[0]; v.y = in[1]; v.z = in[2]; v.w = in[3]; }
    else { v.x = in[0]; v.y = in[1]; }
    *reinterpret_cast<T*>(p) = v;
}

// ---- step prologue (launched at the start of step j, and once with j = k after the loop).
// Finalises index i = j-1 from the reduced accumulators: alpha_i, row i of the Cholesky of
// T (L_ii), g_i = (L^{-1} e_1)_i, then beta_i, the breakdown test (reading A12)
// and the scale 1/beta_i of q_j.  Every thread recomputes the scalars it needs (they only
// depend on state written by earlier launches); block 0 / thread 0 persists them.  The
// same launch streams column i of the cache:
//   Rc[:, i] = (z_i - L_{i,i-1} Rc[:, i-1]) / L_ii ;  a += ||b|| g_i Rc[:, i]      (fp64)
__global__ void step_prologue_kernel(LanczosState st, int k, double tol, int m,
                                     const double* __restrict__ z0, const double* __restrict__ z1,
                                     double* __restrict__ Rc, double* __restrict__ a, int mean_y) {
    pdl_wait();
    int* fl = st.flags;
    const int j = *st.jdev;
    const double* __restrict__ z = ((j - 1) & 1) ? z1 : z0;     // z_{j-1}
    const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
    if (j == 0) {
        if (writer) {
            const double b2 = st.bnorm2[0];
            if (!(b2 > 0.0)) { fl[3] = 1; fl[0] = 1; fl[1] = 0; }
            else st.qscale[0] = 1.0 / sqrt(b2);
        }
        return;
    }
    const int i = j - 1;
    if (fl[1] <= i || fl[2] || fl[3]) return;           // stopped at an earlier step
    const double al = st.alpha_cur[0];
    const double amax = fmax(st.amax_bmax[0], fabs(al));
    const double lsub = i > 0 ? st.Ls[i - 1] : 0.0;
    const double piv = al - lsub * lsub;
    if (!(piv > 0.0)) {
        if (writer) { fl[2] = 1; fl[0] = 1; fl[1] = i; }
        return;
    }
    const double ld = sqrt(piv);
    const double gi = (i == 0) ? 1.0 / ld : -lsub * st.g[i - 1] / ld;
    if (writer) {
        st.alpha[i] = al;
        st.Ld[i] = ld;
        st.g[i] = gi;
        st.amax_bmax[0] = amax;
        if (j == k) {
            fl[0] = 1;
            fl[1] = k;
        } else {
            const double b = sqrt(st.beta2_cur[0]);
            const double bmax = fmax(st.amax_bmax[1], b);
            st.amax_bmax[1] = bmax;
            if (!(b >= tol * (amax + 2.0 * bmax))) {
                fl[0] = 1;
                fl[1] = j;
            } else {
                st.beta[i] = b;
                st.Ls[i] = b / ld;
                st.qscale[j] = 1.0 / b;
            }
        }
    }
    const double ag = sqrt(st.bnorm2[0]) * gi;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
        const double prev = i > 0 ? Rc[(int64_t)(i - 1) * m + p] : 0.0;
        const double v = (z[p] - lsub * prev) / ld;
        Rc[(int64_t)i * m + p] = v;
        if (mean_y) a[p] += ag * v;
    }
}

template <typename V>
__global__ void norm2_kernel(const V* __restrict__ b, int64_t n, double* __restrict__ out) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)b[p];
        acc += v * v;
    }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) atomicAdd(out, acc);
}

// Source vector of a reorthogonalisation pass, rows [p, p+W): pass 0 forms the three-term
// residual r' = r - alpha_j q_j - beta_{j-1} q_{j-1} in fp64; later passes read Q~[:, j+1].
template <typename V>
__device__ __forceinline__ void load_src(const V* __restrict__ Q, int64_t ldq, const V* __restrict__ r,
                                         int from_r, int j, double aj, double bj1, int64_t p,
                                         double out[VecT<V>::W]) {
    constexpr int W = VecT<V>::W;
    V x[W];
    if (from_r) {
        V qa[W], qb[W];
        vload<V>(r + p, x);
        vload<V>(Q + (int64_t)j * ldq + p, qa);
        if (j > 0) vload<V>(Q + (int64_t)(j - 1) * ldq + p, qb);
#pragma unroll
        for (int e = 0; e < W; ++e)
            out[e] = (double)x[e] - aj * (double)qa[e] - (j > 0 ? bj1 * (double)qb[e] : 0.0);
    } else {
        vload<V>(Q + (int64_t)(j + 1) * ldq + p, x);
#pragma unroll
        for (int e = 0; e < W; ++e) out[e] = (double)x[e];
    }
}

// ---- reorthogonalisation dots, column-sweep variant (the update kernel's access pattern):
// every thread holds CPT 16-byte chunks of r' in registers and sweeps the columns in blocks of
// 8; the 8 per-lane partials of a block are reduced across the warp by a butterfly
// reduce-scatter (xor 4, 2, 1: 7 shuffles) plus xor 8, 16, after which lane l holds column
// 8b + (l & 7) summed over the warp; lanes 0..7 park it in shared memory (fp64).
// (trace build: held at the production 32 registers, 8 CTAs per SM)
#ifdef LOVE_TRACE_ON
#define LOVE_DOTS_BOUNDS __launch_bounds__(256, 8)
#else
#define LOVE_DOTS_BOUNDS __launch_bounds__(256)
#endif
template <typename V, int CPT>
__global__ void LOVE_DOTS_BOUNDS reorth_dots_sweep_kernel(const V* __restrict__ Q, int64_t ldq, int k, int pass,
                                                                const V* __restrict__ r, LanczosState st,
                                                                const int* __restrict__ gate) {
    pdl_wait();
    LOVE_TRACE(pass == 0 ? kTrDots0 : kTrDots1, *st.jdev);
    if (sizeof(V) == 8 && st.dgks && pass == 1 && st.flags[7]) return;   // DGKS: the step has advanced
    constexpr int W = VecT<V>::W;
    extern __shared__ __align__(16) double smd[];
    const int j = *st.jdev;
    if (st.flags[0] || j >= k - 1) return;
    if (gate != nullptr && !*gate) return;
    if (sizeof(V) == 8 && st.dgks && pass == 1 && !(st.nrm2[1] < 0.5 * st.nrm2[0])) return;   // DGKS: pass 1 not needed
    const int from_r = pass == 0;
    double* __restrict__ c_out = st.c_cur + ((int64_t)pass * st.crep + blockIdx.x % st.crep) * c_stride(st, k);
    const int ncols = j + 1;
    // column groups (blockIdx.y, small n): this CTA sweeps columns [cbeg, cend) only
    const int cpg = (int)round_up(ceil_div(ncols, gridDim.y), 8);
    const int cbeg = blockIdx.y * cpg, cend = min(ncols, cbeg + cpg);
    if (cbeg >= cend) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* csum = smd;                                   // [nw][ncols]
    const double sj = st.qscale[j];
    const double aj = st.alpha_cur[0] * sj;
    const double bj1 = j > 0 ? st.beta[j - 1] * st.qscale[j - 1] : 0.0;
    const int64_t nvec = ldq / W;
    V src[CPT][W];
    int64_t qv[CPT];
    double s2 = 0.0;                                     // ||r'||^2 partial (DGKS, pass 0, fp64 only)
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
        qv[u] = ((int64_t)blockIdx.x * CPT + u) * blockDim.x + threadIdx.x;
        double v[W];
        if (qv[u] < nvec) load_src<V>(Q, ldq, r, from_r, j, aj, bj1, qv[u] * W, v);
        else
#pragma unroll
            for (int e = 0; e < W; ++e) v[e] = 0.0;
#pragma unroll
        for (int e = 0; e < W; ++e) {
            src[u][e] = (V)v[e];
            if constexpr (sizeof(V) == 8) s2 += v[e] * v[e];
        }
    }
    if constexpr (sizeof(V) == 8) {                     // (the fp32 instantiation keeps 32 registers)
        if (st.dgks && pass == 0 && blockIdx.y == 0) {  // one column group counts the rows once
            __shared__ double red2[32];
            s2 = block_sum(s2, red2);
            if (threadIdx.x == 0) atomicAdd(&st.nrm2[0], s2);
        }
    }
    const int b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1, b0 = lane & 1;
    constexpr int NB = LOVE_SWEEP_NB;                    // 8-column blocks whose loads are issued together
    for (int c00 = cbeg; c00 < cend; c00 += 8 * NB) {
    V pvb[NB][8];
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
            V& pcell = pvb[bb][cc];
            const int cidx = c00 + 8 * bb + cc;
            pcell = V(0);
            if (cidx < cend) {
#pragma unroll
                for (int u = 0; u < CPT; ++u) {
                    if (qv[u] < nvec) {
                        V a[W];
                        vload<V>(Q + (int64_t)cidx * ldq + qv[u] * W, a);
#pragma unroll
                        for (int e = 0; e < W; ++e) pcell += a[e] * src[u][e];
                    }
                }
            }
        }
#pragma unroll
    for (int bb = 0; bb < NB; ++bb) {
        const int c0 = c00 + 8 * bb;
        if (c0 >= cend) break;
        const V* pv = pvb[bb];
        // reduce-scatter: keep 4 of 8 (xor 4), 2 of 4 (xor 2), 1 of 2 (xor 1)
        double h4[4], h2[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double keep = (double)(b2 ? pv[i + 4] : pv[i]), send = (double)(b2 ? pv[i] : pv[i + 4]);
            h4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = b1 ? h4[i + 2] : h4[i], send = b1 ? h4[i] : h4[i + 2];
            h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        double h1;
        {
            const double keep = b0 ? h2[1] : h2[0], send = b0 ? h2[0] : h2[1];
            h1 = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
        h1 += __shfl_xor_sync(0xffffffffu, h1, 8);
        h1 += __shfl_xor_sync(0xffffffffu, h1, 16);
        const int col = c0 + (b2 << 2 | b1 << 1 | b0);
        if (lane < 8 && col < cend) csum[wid * ncols + col] = h1;
    }
    }
    __syncthreads();
    for (int i = cbeg + threadIdx.x; i < cend; i += blockDim.x) {
        double tot = 0.0;
        for (int w = 0; w < nw; ++w) tot += csum[w * ncols + i];
        atomicAdd(&c_out[i], tot * st.qscale[i]);
    }
}

// ---- one-sync step (several GPUs, fp32, probe X9): ONE pass over Q~_j gives
// the three dot vectors c_r = Q_j^T r, g1 = Q_j^T q_j and g2 = Q_j^T q_{j-1} (normalised
// columns) into c_cur[0 .. 3(k+1)), so a single all-reduce replaces those of alpha and of the
// reorthogonalisation dots: alpha_j = c_r[j] and Q_j^T r' = c_r - alpha_j g1 - beta_{j-1} g2
// for the three-term residual r' (reorth_update_kernel, kUpd1Sync).  Same sweep as the kernel
// above (8-column blocks, butterfly reduce-scatter per source, fp64 across lanes); it also
// runs at j = k-1, where only alpha is needed.
template <typename V>
__global__ void __launch_bounds__(256) reorth_dots3_kernel(const V* __restrict__ Q, int64_t ldq, int k,
                                                           const V* __restrict__ r, LanczosState st) {
    pdl_wait();
    LOVE_TRACE(kTrDots0, *st.jdev);
    constexpr int W = VecT<V>::W;
    extern __shared__ __align__(16) double smd[];
    const int j = *st.jdev;
    if (st.flags[0] || j >= k) return;
    const int ncols = j + 1;
    const int cpg = (int)round_up(ceil_div(ncols, gridDim.y), 8);
    const int cbeg = blockIdx.y * cpg, cend = min(ncols, cbeg + cpg);
    if (cbeg >= cend) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t K1 = k + 1;
    double* csum = smd;                                   // [3][nw][ncols]
    const int64_t nvec = ldq / W;
    const int64_t qv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    V src[3][W];
    {
        V a[W], b[W], c[W];
#pragma unroll
        for (int e = 0; e < W; ++e) a[e] = b[e] = c[e] = V(0);
        if (qv < nvec) {
            vload<V>(r + qv * W, a);
            vload<V>(Q + (int64_t)j * ldq + qv * W, b);
            if (j > 0) vload<V>(Q + (int64_t)(j - 1) * ldq + qv * W, c);
        }
#pragma unroll
        for (int e = 0; e < W; ++e) { src[0][e] = a[e]; src[1][e] = b[e]; src[2][e] = c[e]; }
    }
    const int b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1, b0 = lane & 1;
    for (int c0 = cbeg; c0 < cend; c0 += 8) {
        V pv[3][8];
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
            const int cidx = c0 + cc;
#pragma unroll
            for (int sidx = 0; sidx < 3; ++sidx) pv[sidx][cc] = V(0);
            if (cidx < cend && qv < nvec) {
                V a[W];
                vload<V>(Q + (int64_t)cidx * ldq + qv * W, a);
#pragma unroll
                for (int sidx = 0; sidx < 3; ++sidx)
#pragma unroll
                    for (int e = 0; e < W; ++e) pv[sidx][cc] += a[e] * src[sidx][e];
            }
        }
#pragma unroll
        for (int sidx = 0; sidx < 3; ++sidx) {
            double h4[4], h2[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double keep = (double)(b2 ? pv[sidx][i + 4] : pv[sidx][i]);
                const double send = (double)(b2 ? pv[sidx][i] : pv[sidx][i + 4]);
                h4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const double keep = b1 ? h4[i + 2] : h4[i], send = b1 ? h4[i] : h4[i + 2];
                h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
            double h1;
            {
                const double keep = b0 ? h2[1] : h2[0], send = b0 ? h2[0] : h2[1];
                h1 = keep + __shfl_xor_sync(0xffffffffu, send, 1);
            }
            h1 += __shfl_xor_sync(0xffffffffu, h1, 8);
            h1 += __shfl_xor_sync(0xffffffffu, h1, 16);
            const int col = c0 + (b2 << 2 | b1 << 1 | b0);
            if (lane < 8 && col < cend) csum[((int64_t)sidx * nw + wid) * ncols + col] = h1;
        }
    }
    __syncthreads();
    const double sj = st.qscale[j], sj1 = j > 0 ? st.qscale[j - 1] : 0.0;
    const int nc = cend - cbeg;
    for (int e = threadIdx.x; e < 3 * nc; e += blockDim.x) {
        const int sidx = e / nc, i = cbeg + (e - sidx * nc);
        double tot = 0.0;
        for (int w = 0; w < nw; ++w) tot += csum[((int64_t)sidx * nw + w) * ncols + i];
        const double sc = st.qscale[i] * (sidx == 0 ? 1.0 : sidx == 1 ? sj : sj1);
        atomicAdd(&st.c_cur[sidx * K1 + i], tot * sc);
    }
}

// the current step's accumulators back to zero (one thread)
__device__ __forceinline__ void clear_step_acc(const LanczosState& st, int k) {
    st.alpha_cur[0] = 0.0;
    st.beta2_cur[0] = 0.0;
    for (int64_t i = 0; i < st.c_len; ++i) st.c_cur[i] = 0.0;
}

// multi-GPU path: after the prologue has consumed the previous step's accumulators
__global__ void clear_acc_kernel(LanczosState st, int k) {
    pdl_wait();
    if (threadIdx.x == 0 && blockIdx.x == 0) clear_step_acc(st, k);
}

// Scalars of index i once alpha_i and beta_i^2 are complete (same rules as the prologue):
// alpha_i, row i of the Cholesky of T, g_i = (L^{-1} e_1)_i, beta_i, the
// breakdown test (reading A12) and the scale of q_{i+1}.  One thread.
// (returns true when the Lanczos stops here or had stopped).  Every input is loaded before the
// first use: the step's serial tail pays one memory round trip for them, not one per use.
struct FinIn {                                     // finalize_index's inputs other than beta^2
    int f0, f1, f2, f3;
    double al, am0, bm0, lsub, gprev;
};
__device__ __forceinline__ FinIn fin_inputs(const LanczosState& st, int i) {
    const int* fl = st.flags;
    FinIn f;
    f.f0 = fl[0];
    f.f1 = fl[1];
    f.f2 = fl[2];
    f.f3 = fl[3];
    f.al = st.alpha_cur[0];
    f.am0 = st.amax_bmax[0];
    f.bm0 = st.amax_bmax[1];
    f.lsub = (st.chol && i > 0) ? st.Ls[i - 1] : 0.0;
    f.gprev = (st.chol && i > 0) ? st.g[i - 1] : 0.0;
    return f;
}
__device__ __forceinline__ bool finalize_index(const LanczosState& st, int i, int k, double tol, const FinIn& in) {
    int* fl = st.flags;
    const int f0 = in.f0, f1 = in.f1, f2 = in.f2, f3 = in.f3;
    const double al = in.al, am0 = in.am0, bm0 = in.bm0, b2 = st.beta2_cur[0];
    const double lsub = in.lsub, gprev = in.gprev;
    if (f1 <= i || f2 || f3) return f0 != 0;
    const double amax = fmax(am0, fabs(al));
    double ld = 1.0;
    if (st.chol) {                                  // row i of the Cholesky of T
        const double piv = al - lsub * lsub;
        if (!(piv > 0.0)) {
            fl[2] = 1;
            fl[0] = 1;
            fl[1] = i;
            return true;
        }
        ld = sqrt(piv);
        st.Ld[i] = ld;
        st.g[i] = (i == 0) ? 1.0 / ld : -lsub * gprev / ld;
    }
    st.alpha[i] = al;
    st.amax_bmax[0] = amax;
    if (i + 1 == k) {
        fl[0] = 1;
        fl[1] = k;
        return true;
    }
    const double b = sqrt(b2);
    const double bmax = fmax(bm0, b);
    st.amax_bmax[1] = bmax;
    if (!(b >= tol * (amax + 2.0 * bmax))) {
        fl[0] = 1;
        fl[1] = i + 1;
        return true;
    }
    st.beta[i] = b;
    if (st.chol) st.Ls[i] = b / ld;
    st.qscale[i + 1] = 1.0 / b;
    return f0 != 0;
}

// Last-CTA-done step advance (every CTA calls it once at its end): the last CTA optionally
// finalises the scalars of index j (single GPU: beta_j^2 is complete once every CTA of the
// update has added its part) and writes j + 1 to the step index.

// true in the last CTA of the grid to get here (every CTA calls it once)
__device__ __forceinline__ bool last_cta(const LanczosState& st) {
    __shared__ int last;
    __syncthreads();
    LOVE_TRACE_ARRIVE(kTrArrive, *st.jdev);
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned prev = atomicAdd(reinterpret_cast<unsigned*>(st.step_ctr), 1u);
        last = prev == gridDim.x - 1;
        if (last) __threadfence();
    }
    __syncthreads();
    return last != 0;
}

// the last CTA's part of advance_step.  No trailing fence: the next kernel reads these after
// griddepcontrol.wait (the grid has completed and its writes are visible); only the host's
// mapped done flag needs the system fence.
template <bool COND>
__device__ __forceinline__ void advance_finish(const LanczosState& st, int j, bool fin, int k, double tol,
                                               const FinIn& in) {
    if (fin)   // the reorthogonalisation dot accumulators (the scalars do not read them)
        for (int64_t i = threadIdx.x; i < st.c_len; i += blockDim.x) st.c_cur[i] = 0.0;
    if (threadIdx.x == 0) {
        bool done;
        if (fin) {
            done = finalize_index(st, j, k, tol, in);
            st.alpha_cur[0] = 0.0;
            st.beta2_cur[0] = 0.0;
            if (st.nrm2 != nullptr) st.nrm2[0] = st.nrm2[1] = 0.0;
        } else {
            done = st.flags[0] != 0;
        }
        if (st.hdone != nullptr && done) {           // tell the host to stop replaying
            *(volatile int*)st.hdone = 1;
            __threadfence_system();
        }
        LOVE_TRACE(kTrAdvanced, j);
        st.step_ctr[0] = 0;
        st.jdev[0] = j + 1;
        if constexpr (COND) {                        // inside the WHILE graph node (LOVE_COND_STEPS)
            st.flags[6] += 1;
            if (done || j + 1 >= st.cond_limit) cudaGraphSetConditional(st.cond, 0);
        }
    }
}

// (thread 0 loads the scalar inputs before the step counter: their round trip overlaps the fence
// and the counter's)
// COND: the kernel variant launched inside the WHILE graph node; only it carries the
// cudaGraphSetConditional call (ncu does not profile kernels that can set a conditional handle)
template <bool COND>
__device__ __forceinline__ void advance_step(const LanczosState& st, int j, bool fin = false, int k = 0,
                                             double tol = 0.0) {
    FinIn in{};
    if (fin && threadIdx.x == 0) in = fin_inputs(st, j);
    if (last_cta(st)) advance_finish<COND>(st, j, fin, k, tol, in);
}

// DGKS-gated CGS2 (fp64, one GPU): the last CTA of the FIRST pass's update decides.  If
// ||r''||^2 >= ||r'||^2 / 2 the second pass is not needed: beta_j^2 = ||r''||^2 and the step
// advances right here; flags[7] = 1 tells the second pass's two kernels of this step to return
// at once (no grid-wide step counter, no scalars).  Otherwise flags[7] = 0 and the second pass
// runs and advances as before.
template <bool COND>
__device__ __forceinline__ void dgks_decide(const LanczosState& st, int j, bool fin, int k, double tol) {
    FinIn in{};
    if (fin && threadIdx.x == 0) in = fin_inputs(st, j);
    if (!last_cta(st)) return;
    const bool skip = !(st.nrm2[1] < 0.5 * st.nrm2[0]);
    if (!skip) {
        if (threadIdx.x == 0) {
            st.flags[7] = 0;
            st.step_ctr[0] = 0;
        }
        return;
    }
    if (threadIdx.x == 0) {
        st.beta2_cur[0] = st.nrm2[1];
        st.flags[7] = 1;
    }
    __syncthreads();
    advance_finish<COND>(st, j, fin, k, tol, in);
}

// ---- reorthogonalisation update: Q~[:, j+1] = src - sum_i c_i q_i ; beta2 += ||.||^2
// update modes: accumulate beta^2 / advance the step (the step's last kernel) / three-term
// only (no reorthogonalisation columns; partial reorthogonalisation)
constexpr int kUpdBeta = 1, kUpdAdvance = 2, kUpd3T = 4, kUpd1Sync = 8;

template <typename V, int CG = 1, bool COND = false>
__global__ void __launch_bounds__(256) reorth_update_kernel(V* __restrict__ Q, int64_t ldq, int64_t n, int k,
                                                            int pass, int mode, const V* __restrict__ r,
                                                            LanczosState st, double tol, int fold,
                                                            const int* __restrict__ gate) {
    pdl_wait();
    LOVE_TRACE(pass == 0 ? kTrUpdate0 : kTrUpdate1, *st.jdev);
    constexpr int W = VecT<V>::W;
    extern __shared__ double cf[];             // [j+1] coefficient of Q~[:, i], as V
    V* __restrict__ cfv = reinterpret_cast<V*>(cf);
    __shared__ double red[32];
    // DGKS: the first pass's update already advanced the step (dgks_decide)
    if (sizeof(V) == 8 && st.dgks && pass == 1 && st.flags[7]) return;
    const int j = *st.jdev;
    // the last pass's update is the last kernel of step j: its last CTA to finish advances
    // the device step index (every CTA has read j by then), also on the early-exit paths
    if (st.flags[0] || j >= k - 1) {
        if (sizeof(V) == 8 && st.dgks && pass == 0 && blockIdx.x == 0 && threadIdx.x == 0) st.flags[7] = 0;
        // one-sync step: alpha of the last step comes from the dots vector (no gather partials)
        if ((mode & kUpd1Sync) && !st.flags[0] && j == k - 1 && blockIdx.x == 0 && threadIdx.x == 0)
            st.alpha_cur[0] = st.c_cur[j];
        if (mode & kUpdAdvance) advance_step<COND>(st, j, fold && j == k - 1, k, tol);
        return;
    }
    if (gate != nullptr && !*gate) {           // partial: no reorthogonalisation this step
        if (mode & kUpdAdvance) advance_step<COND>(st, j, fold != 0, k, tol);
        return;
    }
    if (sizeof(V) == 8 && st.dgks && pass == 1 && !(st.nrm2[1] < 0.5 * st.nrm2[0])) {
        // DGKS: the first pass kept ||r''|| >= ||r'|| / sqrt 2, the column stands; beta^2 is its norm
        if (threadIdx.x == 0) st.beta2_cur[0] = st.nrm2[1];
        if (mode & kUpdAdvance) advance_step<COND>(st, j, fold != 0, k, tol);
        return;
    }
    const int from_r = pass == 0;
    const int64_t cst = c_stride(st, k);
    const double* __restrict__ c_in = st.c_cur + (int64_t)pass * st.crep * cst;
    double* __restrict__ beta2_out =
        (mode & kUpdBeta) ? st.beta2_cur : (sizeof(V) == 8 && st.dgks && pass == 0) ? st.nrm2 + 1 : nullptr;
    const int ncols = (mode & kUpd3T) ? 0 : j + 1;
    // one-sync step: alpha_j = c_r[j], coefficients of r' = r - alpha q_j - beta q_{j-1}:
    // Q_j^T r' = c_r - alpha_j g1 - beta_{j-1} g2 (all-reduced, normalised columns)
    const double al1 = (mode & kUpd1Sync) ? c_in[j] : 0.0;
    const double bt1 = (mode & kUpd1Sync) && j > 0 ? st.beta[j - 1] : 0.0;
    if ((mode & kUpd1Sync) && blockIdx.x == 0 && threadIdx.x == 0) st.alpha_cur[0] = al1;
    for (int i = threadIdx.x; i < ncols; i += blockDim.x) {
        double ci;
        if (mode & kUpd1Sync) {
            ci = c_in[i] - al1 * c_in[cst + i] - bt1 * c_in[2 * cst + i];
        } else if (st.crep == 4) {              // independent loads (one L2 round trip)
            ci = (c_in[i] + c_in[cst + i]) + (c_in[2 * cst + i] + c_in[3 * cst + i]);
        } else {
            ci = 0.0;
            for (int rp = 0; rp < st.crep; ++rp) ci += c_in[rp * cst + i];
        }
        cfv[i] = (V)(ci * st.qscale[i]);       // rounded to V once per CTA, not per column
    }
    __syncthreads();
    const double sj = st.qscale[j];
    const double aj = ((mode & kUpd1Sync) ? al1 : st.alpha_cur[0]) * sj;
    const double bj1 = j > 0 ? st.beta[j - 1] * st.qscale[j - 1] : 0.0;
    double b2 = 0.0;
    const int64_t nchunks = ldq / W;
    if constexpr (CG > 1) {
        // small n (few chunks, long column sweeps): CG groups of 256 / CG threads share each
        // chunk group, group g sweeping a contiguous 1/CG of the columns; the partial sums meet
        // in shared memory and group 0 finishes the chunk
        constexpr int T = 256 / CG;
        using VT = typename VecT<V>::T;
        __shared__ VT part[CG - 1][T];
        const int grp = threadIdx.x / T, t = threadIdx.x % T;
        const int per = (ncols + CG - 1) / CG;
        const int cbeg = min(ncols, grp * per), cend = min(ncols, cbeg + per);
        for (int64_t q0 = blockIdx.x * (int64_t)T; q0 < nchunks; q0 += (int64_t)gridDim.x * T) {
            const int64_t q = q0 + t;
            const bool live = q < nchunks;
            const int64_t p = q * W;
            V acc[W];
#pragma unroll
            for (int e = 0; e < W; ++e) acc[e] = V(0);
            if (live && cend > cbeg) {
                const V* col = Q + (int64_t)(cend - 1) * ldq + p;
                int i = cend - 1;
                for (; i >= cbeg + kUpdB - 1; i -= kUpdB) {
                    V a[kUpdB][W];
#pragma unroll
                    for (int u = 0; u < kUpdB; ++u) vload<V>(col - (int64_t)u * ldq, a[u]);
#pragma unroll
                    for (int u = 0; u < kUpdB; ++u) {
                        const V ci = cfv[i - u];
#pragma unroll
                        for (int e = 0; e < W; ++e) acc[e] += ci * a[u][e];
                    }
                    col -= (int64_t)kUpdB * ldq;
                }
                for (; i >= cbeg; --i) {
                    V a[W];
                    vload<V>(col, a);
                    const V ci = cfv[i];
#pragma unroll
                    for (int e = 0; e < W; ++e) acc[e] += ci * a[e];
                    col -= ldq;
                }
            }
            if (grp > 0) vstore<V>(reinterpret_cast<V*>(&part[grp - 1][t]), acc);
            __syncthreads();
            if (grp == 0 && live) {
#pragma unroll
                for (int h = 0; h < CG - 1; ++h) {
                    V o2[W];
                    vload<V>(reinterpret_cast<const V*>(&part[h][t]), o2);
#pragma unroll
                    for (int e = 0; e < W; ++e) acc[e] += o2[e];
                }
                double v[W];
                load_src<V>(Q, ldq, r, from_r, j, aj, bj1, p, v);
                V o[W];
#pragma unroll
                for (int e = 0; e < W; ++e) {
                    o[e] = (p + e < n) ? (V)(v[e] - (double)acc[e]) : V(0);
                    b2 += (double)o[e] * (double)o[e];
                }
                vstore<V>(Q + (int64_t)(j + 1) * ldq + p, o);
            }
            __syncthreads();
        }
    } else {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nchunks;
             q += (int64_t)gridDim.x * blockDim.x) {
            const int64_t p = q * W;
            double v[W];
            load_src<V>(Q, ldq, r, from_r, j, aj, bj1, p, v);
            V acc[W];
#pragma unroll
            for (int e = 0; e < W; ++e) acc[e] = V(0);
            // columns are swept LAST to first: the dots pass streamed Q~ from column 0 up, so its
            // last columns are the ones still in L2; the next step's dots pass starts at column
            // 0, the one this pass reads last.
            // batches of kUpdB columns: all kUpdB 16-byte loads are issued before the first FMA
            // (same summation order as one column at a time)
            const V* col = Q + (int64_t)(ncols - 1) * ldq + p;
            int i = ncols - 1;
            for (; i >= kUpdB - 1; i -= kUpdB) {
                V a[kUpdB][W];
#pragma unroll
                for (int u = 0; u < kUpdB; ++u) vload<V>(col - (int64_t)u * ldq, a[u]);
#pragma unroll
                for (int u = 0; u < kUpdB; ++u) {
                    const V ci = cfv[i - u];
#pragma unroll
                    for (int e = 0; e < W; ++e) acc[e] += ci * a[u][e];
                }
                col -= (int64_t)kUpdB * ldq;
            }
            for (; i >= 0; --i) {
                V a[W];
                vload<V>(col, a);
                const V ci = cfv[i];
#pragma unroll
                for (int e = 0; e < W; ++e) acc[e] += ci * a[e];
                col -= ldq;
            }
            V o[W];
#pragma unroll
            for (int e = 0; e < W; ++e) {
                o[e] = (p + e < n) ? (V)(v[e] - (double)acc[e]) : V(0);
                b2 += (double)o[e] * (double)o[e];
            }
            vstore<V>(Q + (int64_t)(j + 1) * ldq + p, o);
        }
    }
    if (beta2_out != nullptr) {
        b2 = block_sum(b2, red);
        if (threadIdx.x == 0) atomicAdd(beta2_out, b2);
    }
    if (mode & kUpdAdvance) advance_step<COND>(st, j, fold != 0, k, tol);
    if constexpr (sizeof(V) == 8) {
        if (st.dgks == 2 && pass == 0 && !(mode & kUpdAdvance)) dgks_decide<COND>(st, j, fold != 0, k, tol);
    }
}

// Rc (fp64, m x k_eff column-major) -> V, m x k_pad row-major (zero padded)
template <typename V>
__global__ void rc_transpose_kernel(const double* __restrict__ Rcc, int m, int k_eff, int k_pad,
                                    V* __restrict__ Rc) {
    __shared__ double tile[32][33];
    const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int col = c0 + y, p = p0 + threadIdx.x;
        tile[y][threadIdx.x] = (col < k_eff && p < m) ? Rcc[(int64_t)col * m + p] : 0.0;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int p = p0 + y, col = c0 + threadIdx.x;
        if (p < m && col < k_pad) Rc[(int64_t)p * k_pad + col] = (V)tile[threadIdx.x][y];
    }
}




// ---- partial reorthogonalisation.  Simon's recurrence
// estimates omega_{j+1,i} ~ q_{j+1}^T q_i from T alone, after the three-term vector
// r' = r - alpha_j q_j - beta_{j-1} q_{j-1} and its norm beta_j (three-term) are known:
//   beta_j omega_{j+1,i} = beta_i omega_{j,i+1} + (alpha_i - alpha_j) omega_{j,i}
//                          + beta_{i-1} omega_{j,i-1} - beta_{j-1} omega_{j-1,i}  +/- eps (beta_i + beta_j)
//   omega_{j+1,j} = eps, omega_{j+1,j+1} = 1.
// If max_i |omega_{j+1,i}| > tol, q~_{j+1} gets one CGS pass against Q_j (and so does the
// next vector); the estimates of both rows are then reset to eps.  omega rows rotate over
// three slots: row j lives in slot j % 3.
__global__ void __launch_bounds__(256) pro_decide_kernel(LanczosState st, int k) {
    pdl_wait();
    __shared__ double red[32];
    __shared__ int reo;
    const int j = *st.jdev;
    if (st.flags[0] || j >= k - 1) {
        if (threadIdx.x == 0) st.pro[0] = 0;
        return;
    }
    const double eps = st.pro_eps;
    const double bj = sqrt(st.beta2_cur[0]);
    const double aj = st.alpha_cur[0];
    const double bjm1 = j > 0 ? st.beta[j - 1] : 0.0;
    const int64_t ld = k + 1;
    double* __restrict__ wp = st.omega + ((j + 2) % 3) * ld;    // row j - 1
    double* __restrict__ wc = st.omega + (j % 3) * ld;          // row j
    double* __restrict__ wn = st.omega + ((j + 1) % 3) * ld;    // row j + 1
    double mx = 0.0;
    for (int i = threadIdx.x; i < j; i += blockDim.x) {
        double t = st.beta[i] * wc[i + 1] + (st.alpha[i] - aj) * wc[i] - bjm1 * wp[i];
        if (i > 0) t += st.beta[i - 1] * wc[i - 1];
        const double w = (t + copysign(eps * (st.beta[i] + bj), t)) / bj;
        wn[i] = w;
        mx = fmax(mx, fabs(w));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        const int force = st.pro[1];
        const int r = force || !(m <= st.pro_tol) || !(bj > 0.0);
        reo = r;
        st.pro[0] = r;
        st.pro[1] = r ? !force : 0;
        if (r) {
            st.pro[2] += 1;
            st.beta2_cur[0] = 0.0;       // the reorthogonalising update recomputes beta_j^2
        }
    }
    __syncthreads();
    if (reo) {
        for (int i = threadIdx.x; i <= j; i += blockDim.x) wn[i] = eps;
        for (int i = threadIdx.x; i < j; i += blockDim.x) wc[i] = eps;
    } else if (threadIdx.x == 0) {
        wn[j] = eps;
    }
    if (threadIdx.x == 0) wn[j + 1] = 1.0;
}

// q_0 = b / ||b|| (scale of column 0) or the zero-probe flag (folded-prologue path)
__global__ void init_q0_kernel(LanczosState st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double b2 = st.bnorm2[0];
    if (!(b2 > 0.0)) {
        st.flags[3] = 1;
        st.flags[0] = 1;
        st.flags[1] = 0;
    } else {
        st.qscale[0] = 1.0 / sqrt(b2);
    }
}

// the last streamed cache column (index *jdev - 1) after the loop
__global__ void stream_rc_kernel(RcStream rs) {
    pdl_wait();
    stream_rc_column(rs, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

template <typename V>
// launch of reorth_update_kernel<V, CG, COND> for a runtime CG in {1, 2, 4}; COND when the step
// runs inside the WHILE graph node (st.cond set)
#define LOVE_UPDATE(V_, cg_, cond_, grid_, smem_, stream_, ...)                                                 \
    do {                                                                                                        \
        if (cond_) {                                                                                            \
            if ((cg_) == 4) LOVE_LAUNCH((reorth_update_kernel<V_, 4, true>), grid_, 256, smem_, stream_, __VA_ARGS__); \
            else if ((cg_) == 2) LOVE_LAUNCH((reorth_update_kernel<V_, 2, true>), grid_, 256, smem_, stream_, __VA_ARGS__); \
            else LOVE_LAUNCH((reorth_update_kernel<V_, 1, true>), grid_, 256, smem_, stream_, __VA_ARGS__);     \
        } else {                                                                                                \
            if ((cg_) == 4) LOVE_LAUNCH((reorth_update_kernel<V_, 4>), grid_, 256, smem_, stream_, __VA_ARGS__); \
            else if ((cg_) == 2) LOVE_LAUNCH((reorth_update_kernel<V_, 2>), grid_, 256, smem_, stream_, __VA_ARGS__); \
            else LOVE_LAUNCH((reorth_update_kernel<V_, 1>), grid_, 256, smem_, stream_, __VA_ARGS__);           \
        }                                                                                                       \
    } while (0)

struct StepPlan {
    Cache* c;
    int k, m, P, mean_y, gm, gu;
    int ucg = 1;                  // column groups per CTA of the update (update_groups)
    bool fold;                    // single GPU: scalars in the update's last CTA, cache column in the gather
    RcStream rs;
    bool mfuse;                   // d = 1, one GPU: the FFT's first pass reads the scatter moments
    bool pfuse3 = false;          // d = 3 fp32, one GPU: the first axis product reads the last-axis sums
    bool partial;                 // partial reorthogonalisation (single GPU)
    bool one_sync;                // several GPUs, fp32, one CGS pass: the one-sync step (reorth_dots3)
    int64_t ldq;
    size_t smu;
};

// Enqueue one Lanczos step (the step index lives in device memory).  j_host only picks the
// z buffer of the step (z_j alternates between two buffers).
// dots grid: one CTA per 256 row chunks, and column groups when that leaves the GPU idle
inline dim3 dots_grid(int64_t ldq, int W, int k) {
    const int gx = (int)ceil_div(ldq / W, 256);
    // column groups fill the GPU up to `target` CTAs, 4 per SM (2 per SM: cfg5 4.78 vs 4.70 ms,
    // cfg3 7.90 vs 7.81 ms; 8 per SM between them; LOVE_DOTS_TARGET overrides)
    static const int target = std::getenv("LOVE_DOTS_TARGET") ? std::atoi(std::getenv("LOVE_DOTS_TARGET")) : 148 * 4;
    const int cg = std::max(1, std::min({16, target / std::max(gx, 1), (k + 7) / 8}));
    return dim3((unsigned)gx, (unsigned)cg);
}

template <typename V>
void enqueue_step(const StepPlan<V>& pl, int j_host, cudaStream_t s) {
    Cache& c = *pl.c;
    const LanczosState& st = c.st;
    V* Q = (V*)c.Q;
    V* r = (V*)c.r;
    double* u = (double*)c.u;
    const StepRef ref{st.jdev, pl.ldq, st.qscale, st.flags};
    if (!pl.fold) {
        ProfScope ps(LOVE_PROF_SCALARS, s);
        LOVE_LAUNCH(step_prologue_kernel, pl.gm, 256, 0, s, st, pl.k, c.tol, pl.m, (const double*)c.z[0],
                    (const double*)c.z[1], (double*)c.Rc_col, (double*)c.a, pl.mean_y);
        LOVE_LAUNCH(clear_acc_kernel, 1, 32, 0, s, st, pl.k);
    }
    {
        ProfScope ps(LOVE_PROF_SCATTER, s);
        launch_scatter<V>(c, Q, ref, u, s, pl.mfuse || pl.pfuse3);
    }
    if (c.comm != nullptr) {
        ProfScope ps(LOVE_PROF_COMM, s);
        allreduce_sum(c, u, pl.m, true, s);
    }
    double* zj = (double*)c.z[j_host & 1];
    {
        ProfScope ps(LOVE_PROF_KUU, s);
        DoneScope ds(st.flags);
        launch_kuu(c, u, zj, s, pl.mfuse ? (const double*)c.Mc : nullptr, pl.pfuse3 ? &ref : nullptr);
    }
    {
        ProfScope ps(LOVE_PROF_GATHER, s);
        launch_gather<V>(c, zj, Q, ref, r, pl.one_sync ? nullptr : st.alpha_cur, s, pl.fold ? &pl.rs : nullptr);
    }
    if (pl.one_sync) {
        // one pass over Q~_j, one all-reduce of the three dot vectors (alpha included), the
        // update, the beta^2 all-reduce: three collectives per step instead of four
        {
            ProfScope ps(LOVE_PROF_REORTH_DOTS, s);
            LOVE_LAUNCH(reorth_dots3_kernel<V>, dots_grid(pl.ldq, VecT<V>::W, pl.k), 256,
                        sizeof(double) * 3 * 8 * (pl.k + 1), s, (const V*)Q, pl.ldq, pl.k, (const V*)r, st);
        }
        {
            ProfScope ps(LOVE_PROF_COMM, s);
            allreduce_sum(c, st.c_cur, 3 * (int64_t)(pl.k + 1), true, s);
        }
        {
            ProfScope ps(LOVE_PROF_REORTH_UPDATE, s);
            LOVE_UPDATE(V, pl.ucg, st.cond != 0, pl.gu, pl.smu, s, Q, pl.ldq, c.n, pl.k, 0,
                        kUpdBeta | kUpdAdvance | kUpd1Sync, r, st, c.tol, 0, (const int*)nullptr);
        }
        {
            ProfScope ps(LOVE_PROF_COMM, s);
            allreduce_sum(c, st.beta2_cur, 1, true, s);
        }
        return;
    }
    if (c.comm != nullptr) {
        ProfScope ps(LOVE_PROF_COMM, s);
        allreduce_sum(c, st.alpha_cur, 1, true, s);
    }
    if (pl.partial) {
        // three-term vector and its norm, the omega recurrence, then (gated) one CGS pass of
        // q~_{j+1} against Q_j whose update finalises the step
        {
            ProfScope ps(LOVE_PROF_REORTH_UPDATE, s);
            LOVE_UPDATE(V, pl.ucg, st.cond != 0, pl.gu, pl.smu, s, Q, pl.ldq, c.n, pl.k, 0, kUpdBeta | kUpd3T, r,
                        st, c.tol, 1, (const int*)nullptr);
        }
        {
            ProfScope ps(LOVE_PROF_SCALARS, s);
            LOVE_LAUNCH(pro_decide_kernel, 1, 256, 0, s, st, pl.k);
        }
        {
            ProfScope ps(LOVE_PROF_REORTH_DOTS, s);
            LOVE_LAUNCH((reorth_dots_sweep_kernel<V, 1>), dots_grid(pl.ldq, VecT<V>::W, pl.k), 256,
                        sizeof(double) * 8 * (pl.k + 1), s, Q, pl.ldq, pl.k, 1, r, st, (const int*)st.pro);
        }
        {
            ProfScope ps(LOVE_PROF_REORTH_UPDATE, s);
            LOVE_UPDATE(V, pl.ucg, st.cond != 0, pl.gu, pl.smu, s, Q, pl.ldq, c.n, pl.k, 1,
                        kUpdBeta | kUpdAdvance, r, st, c.tol, 1, (const int*)st.pro);
        }
        return;
    }
    for (int pass = 0; pass < pl.P; ++pass) {
        {
            ProfScope ps(LOVE_PROF_REORTH_DOTS, s);
            LOVE_LAUNCH((reorth_dots_sweep_kernel<V, 1>), dots_grid(pl.ldq, VecT<V>::W, pl.k), 256,
                        sizeof(double) * 8 * (pl.k + 1), s, Q, pl.ldq, pl.k, pass, r, st, (const int*)nullptr);
        }
        if (c.comm != nullptr) {
            ProfScope ps(LOVE_PROF_COMM, s);
            allreduce_sum(c, st.c_cur + (int64_t)pass * (pl.k + 1), pl.k + 1, true, s);
        }
        {
            ProfScope ps(LOVE_PROF_REORTH_UPDATE, s);
            LOVE_UPDATE(V, pl.ucg, st.cond != 0, pl.gu, pl.smu, s, Q, pl.ldq, c.n, pl.k, pass,
                        pass == pl.P - 1 ? kUpdBeta | kUpdAdvance : 0, r, st, c.tol, pl.fold ? 1 : 0,
                        (const int*)nullptr);
        }
    }
    if (c.comm != nullptr) {
        ProfScope ps(LOVE_PROF_COMM, s);
        allreduce_sum(c, st.beta2_cur, 1, true, s);
    }
}

template <typename V>
void lanczos_impl(Cache& c, cudaStream_t s) {
    StepPlan<V> pl;
    pl.c = &c;
    pl.k = c.k_req;
    pl.m = c.g.m_total;
    pl.P = c.reorth_passes;
    pl.mean_y = c.probe == LOVE_PROBE_Y;
    pl.mfuse = c.Mc != nullptr && c.comm == nullptr;
    pl.pfuse3 = sizeof(V) == 4 && fuse_pull3(c);
    pl.fold = c.comm == nullptr && std::getenv("LOVE_NO_FOLD") == nullptr;
    pl.partial = c.partial;
    // the one-sync step needs 3 (k+1) fp64 partial dots per warp in shared memory
    pl.one_sync = c.comm != nullptr && c.precision == LOVE_FP32 && c.reorth_passes == 1 && !c.partial &&
                  sizeof(double) * 3 * 8 * (size_t)(c.k_req + 1) <= 200 * 1024 &&
                  std::getenv("LOVE_NO_ONE_SYNC") == nullptr;
    if (pl.one_sync) ensure_smem((const void*)reorth_dots3_kernel<V>, sizeof(double) * 3 * 8 * (c.k_req + 1));
    pl.rs = RcStream{c.st, (const double*)c.z[0], (const double*)c.z[1], (double*)c.Rc_col, (double*)c.a, pl.m,
                     pl.mean_y};
    pl.ldq = c.ldq;
    pl.gm = (int)std::min<int64_t>(ceil_div(pl.m, 256), 148 * 8);
    pl.ucg = update_groups(c.ldq / VecT<V>::W);
    pl.gu = update_grid<V>(c.ldq / VecT<V>::W, sizeof(double) * (pl.k + 1), pl.ucg);
    pl.smu = sizeof(double) * (pl.k + 1);
    ensure_smem((const void*)reorth_dots_sweep_kernel<V, 1>, sizeof(double) * 8 * (pl.k + 1));

    host_mark("plan");
    const LanczosState& st = c.st;
    {
        ProfScope ps(LOVE_PROF_SETUP, s);
        LOVE_LAUNCH(norm2_kernel<V>, (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(c.n, 256), 148 * 4)),
                    256, 0, s, (const V*)c.Q, c.n, st.bnorm2);
    }
    if (c.comm != nullptr) {
        ProfScope ps(LOVE_PROF_COMM, s);
        allreduce_sum(c, st.bnorm2, 1, true, s);
    }
    if (pl.fold) {
        ProfScope ps(LOVE_PROF_SCALARS, s);
        LOVE_LAUNCH(init_q0_kernel, 1, 32, 0, s, st);
    }
    trace_begin(c, pl.k, s);
    // the step graph is also captured on several GPUs: its all-reduces have fixed addresses
    const bool graph = !profiling() && std::getenv("LOVE_NO_GRAPH") == nullptr;
    // one GPU: early stop of the replays at breakdown (the device sets a mapped host flag; on
    // several GPUs every rank must issue the same collectives, so they replay to k)
    std::unique_ptr<ReplayThrottle> thr;
    host_mark("q0");
    if (graph && c.comm == nullptr && pl.fold) {
        thr.reset(new ReplayThrottle(c.device));
        c.st.hdone = thr->d;
        pl.rs.st = c.st;
    }
    // every kernel of a step starts with pdl_wait(): its launch can overlap the previous
    // kernel's drain (programmatic dependent launch)
    PdlScope pdl(std::getenv("LOVE_NO_PDL") == nullptr);
    // Opt-in (LOVE_COND_STEPS=G): measured, the WHILE node's per-iteration cost (~6 us) and the
    // host-side instantiation of its body outweigh the launches it saves unless the Lanczos
    // breaks down well before k (cfg5: 2.58 -> 1.91 ms; cfg2: +0.3 ms at G = 2).
    const char* ge_env = std::getenv("LOVE_COND_STEPS");
    int G = ge_env ? std::atoi(ge_env) : kCondSteps;
    G = std::max(2, G - (G & 1));
    if (graph && c.comm == nullptr && ge_env != nullptr && pl.k >= G) {
        // one GPU: a CUDA graph WHILE node whose body is G steps (G even: z buffer parity);
        // the last update of a step clears the condition on breakdown or at the last full
        // body, so the host never polls and at most G - 1 early-exiting steps run past a
        // breakdown (every step kernel returns at once once the Lanczos is done)
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        cuda_check(cudaGraphCreate(&g, 0), "graph create");
        cudaGraphConditionalHandle h;
        cuda_check(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault), "conditional handle");
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        cuda_check(cudaGraphAddNode(&node, g, nullptr, 0, &cp), "conditional node");
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        StepPlan<V> pc = pl;
        LanczosState& cst = c.st;
        cst.cond = (unsigned long long)h;
        const int limit = pl.k - pl.k % G;
        cst.cond_limit = limit;
        pc.rs.st = cst;
        const int64_t before = g_launch_count.load();
        cuda_check(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
                   "begin capture");
        for (int jj = 0; jj < G; ++jj) enqueue_step<V>(pc, jj, s);
        cuda_check(cudaStreamEndCapture(s, &body), "end capture");
        cst.cond = 0;                               // launches after the loop: plain steps
        cst.cond_limit = 0;
        c.cond_nodes = g_launch_count.load() - before;
        c.cond_steps = G;
        g_launch_count -= c.cond_nodes;             // counted after the build from flags[6]
        cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
        cuda_check(cudaGraphLaunch(ge, s), "graph launch");
        for (int j = limit; j < pl.k; ++j) enqueue_step<V>(pl, j, s);
        cuda_check(cudaGraphExecDestroy(ge), "graph destroy");
        cuda_check(cudaGraphDestroy(g), "graph destroy");
    } else if (graph) {
        // one step as a CUDA graph, replayed k times (z buffer parity alternates: capture
        // two steps so both parities are covered and replay the pair)
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        const int64_t before = g_launch_count.load();      // captured launches run once per replay
        host_mark("pre_capture");
        cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
        enqueue_step<V>(pl, 0, s);
        enqueue_step<V>(pl, 1, s);
        cuda_check(cudaStreamEndCapture(s, &g), "end capture");
        host_mark("capture");
        // one GPU: the exec is cached across builds of the same shape (several GPUs: the graph
        // holds NCCL kernels of a per-build communicator, instantiated fresh)
        const bool cache_ge = c.comm == nullptr;
        const std::string key = "lanczos/" + std::to_string(sizeof(V)) + "/" + std::to_string(c.g.d) + "/" +
                                std::to_string(pl.P) + "/" + std::to_string((int)pl.partial) + "/" +
                                std::to_string((int)pl.mfuse) + "/" + std::to_string(pl.ucg);
        if (cache_ge) ge = graph_exec_cached(g, key);
        else cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
        host_mark("instantiate");
        const int64_t nodes = g_launch_count.load() - before;
        g_launch_count -= nodes;
        // replays past a breakdown would only run early-exiting kernels: the host stops as soon
        // as the mapped done flag is set, keeping a window of replays in flight (no stream sync)
        bool stop = false;
        for (int j = 0, i = 0; j + 1 < pl.k; j += 2, ++i) {
            if (thr != nullptr && !thr->admit(i)) {
                stop = true;
                break;
            }
            cuda_check(cudaGraphLaunch(ge, s), "graph launch");
            g_launch_count += nodes;
            if (thr != nullptr) thr->launched(i, s);
        }
        if ((pl.k & 1) && !stop) enqueue_step<V>(pl, pl.k - 1, s);
        if (!cache_ge) cuda_check(cudaGraphExecDestroy(ge), "graph destroy");
        cuda_check(cudaGraphDestroy(g), "graph destroy");
    } else {
        for (int j = 0; j < pl.k; ++j) enqueue_step<V>(pl, j, s);
    }
    c.st.hdone = nullptr;
    if (c.trace != nullptr) trace_end(s);
    if (pl.fold) {   // the last streamed column (its scalars were finalised by the last update)
        ProfScope ps(LOVE_PROF_SCALARS, s);
        LOVE_LAUNCH(stream_rc_kernel, pl.gm, 256, 0, s, pl.rs);
    } else {         // finalise index k-1: alpha_{k-1}, L_{k-1,k-1}, Rc[:, k-1], a
        ProfScope ps(LOVE_PROF_SCALARS, s);
        LOVE_LAUNCH(step_prologue_kernel, pl.gm, 256, 0, s, st, pl.k, c.tol, pl.m, (const double*)c.z[0],
                    (const double*)c.z[1], (double*)c.Rc_col, (double*)c.a, pl.mean_y);
    }
}

__global__ void fill_kernel(double* __restrict__ u, int m, double v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) u[i] = v;
}

// d[i] += sum_p Q~[p, i] y[p] over this CTA's row tile, i < ncols (fp64 accumulation)
template <typename V>
__global__ void __launch_bounds__(256) qty_kernel(const V* __restrict__ Q, int64_t ldq, int64_t n, int ncols,
                                                  const V* __restrict__ y, int64_t tile_rows,
                                                  double* __restrict__ d) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * tile_rows;
    const int64_t r1 = min(n, r0 + tile_rows);
    for (int i = wid; i < ncols; i += nw) {
        const V* __restrict__ q = Q + (int64_t)i * ldq;
        double acc = 0.0;
        for (int64_t p = r0 + lane; p < r1; p += 32) acc += (double)q[p] * (double)y[p];
        acc = warp_sum(acc);
        if (lane == 0) atomicAdd(&d[i], acc);
    }
}

// g = L^{-1} (S d), S = diag(qscale): forward substitution with the bidiagonal factor of T
// (P:295-298), one thread
__global__ void eq4_solve_kernel(LanczosState st, int k_eff, double* __restrict__ d) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double prev = 0.0;
    for (int i = 0; i < k_eff; ++i) {
        const double rhs = d[i] * st.qscale[i] - (i > 0 ? st.Ls[i - 1] * prev : 0.0);
        prev = rhs / st.Ld[i];
        d[i] = prev;
    }
}

// a[p] = sum_i Rc[p, i] g[i]   (Rc column-major fp64, m x k_eff)
__global__ void rc_gemv_kernel(const double* __restrict__ Rc, int m, int k_eff, const double* __restrict__ g,
                               double* __restrict__ a) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int i = 0; i < k_eff; ++i) acc += Rc[(int64_t)i * m + p] * g[i];
        a[p] = acc;
    }
}

template <typename V>
void avgcol_impl(Cache& c, cudaStream_t s) {
    const int m = c.g.m_total;
    double* u = (double*)c.u;
    double* z = (double*)c.z[1];
    double* zero = (double*)dalloc(c, sizeof(double), s);
    LOVE_LAUNCH(fill_kernel, (int)std::min<int64_t>(ceil_div(m, 256), 148 * 8), 256, 0, s, u, m, 1.0 / m);
    launch_kuu(c, u, z, s);
    // r = W^T z + sigma^2 * 0 * r : the gather with a zero scale on its q term
    const StepRef ref{nullptr, 0, zero, nullptr};
    launch_gather<V>(c, z, (const V*)c.r, ref, (V*)c.Q, nullptr, s);
}

template <typename V>
void eq4_impl(Cache& c, cudaStream_t s) {
    const int m = c.g.m_total, ke = c.k_eff;
    double* d = (double*)dalloc(c, sizeof(double) * std::max(ke, 1), s);
    const int64_t tile = std::max<int64_t>(1024, round_up(ceil_div(c.n, 148 * 4), 32));
    if (c.n > 0)
        LOVE_LAUNCH(qty_kernel<V>, (int)ceil_div(c.n, tile), 256, 0, s, (const V*)c.Q, c.ldq, c.n, ke,
                    (const V*)c.ysort, tile, d);
    if (c.comm != nullptr) allreduce_sum(c, d, ke, true, s);
    LOVE_LAUNCH(eq4_solve_kernel, 1, 32, 0, s, c.st, ke, d);
    LOVE_LAUNCH(rc_gemv_kernel, (int)std::min<int64_t>(ceil_div(m, 256), 148 * 8), 256, 0, s,
                (const double*)c.Rc_col, m, ke, d, (double*)c.a);
}

}  // namespace

// One CGS pass of the reorthogonalisation of step *st.jdev on an fp64 basis (used by the
// sampling-cache Lanczos, sample.cu): dots then update; the last pass's update finalises
// the step's scalars (no Cholesky when st.chol == 0) and advances the step index.
void launch_reorth_pass_f64(const LanczosState& st, double* Q, int64_t ldq, int64_t n, int k, int pass,
                            int last_pass, const double* r, double tol, cudaStream_t s) {
    const size_t smd = sizeof(double) * 8 * (k + 1);
    ensure_smem((const void*)reorth_dots_sweep_kernel<double, 1>, smd);
    LOVE_LAUNCH((reorth_dots_sweep_kernel<double, 1>), dots_grid(ldq, 2, k), 256, smd, s, (const double*)Q, ldq,
                k, pass, r, st, (const int*)nullptr);
    const int ucg = update_groups(ldq / 2);
    const int gu = update_grid<double>(ldq / 2, sizeof(double) * (k + 1), ucg);
    const size_t smu = sizeof(double) * (k + 1);

    LOVE_UPDATE(double, ucg, st.cond != 0, gu, smu, s, Q, ldq, n, k, pass,
                last_pass ? kUpdBeta | kUpdAdvance : 0, r, st, tol, 1, (const int*)nullptr);
}

void launch_init_q0(const LanczosState& st, cudaStream_t s) { LOVE_LAUNCH(init_q0_kernel, 1, 32, 0, s, st); }

// CTAs of the reorthogonalisation update for nchunks 16-byte chunks: one per chunk of 256
// threads, capped at the CTAs resident on the GPU at once (a persistent grid-stride launch:
// measured, cfg2 build 11.25 -> 10.95 ms against the 1.65-wave grid; LOVE_UPD_GRID overrides)
// Column groups of the update for nchunks 16-byte chunks: small n runs few, long per-thread
// column sweeps on few SMs; splitting the columns over 2 / 4 thread groups shortens them
// (LOVE_UPD_CG overrides).  Measured: cfg5's sampling Lanczos (m = 10^4: 5000 chunks) and
// main Lanczos (n = 10^5 fp64: 5 10^4 chunks); cfg2-4 (>= 1.25 10^5 chunks) keep one group.
int update_groups(int64_t nchunks) {
    if (const char* e = std::getenv("LOVE_UPD_CG")) {
        const int v = std::atoi(e);
        return v == 2 || v == 4 ? v : 1;
    }
    return nchunks <= 16384 ? 4 : nchunks <= 65536 ? 2 : 1;
}

// CTAs of the update: one per 256 / cg chunks, capped at the CTAs resident on the GPU at once
// (a persistent grid-stride launch: measured, cfg2 build 11.25 -> 10.95 ms against the
// 1.65-wave grid; LOVE_UPD_GRID overrides).  Also raises the kernel's shared-memory limit.
template <typename V>
int update_grid(int64_t nchunks, size_t smem, int cg) {
    const void* fn = cg == 4 ? (const void*)reorth_update_kernel<V, 4>
                   : cg == 2 ? (const void*)reorth_update_kernel<V, 2> : (const void*)reorth_update_kernel<V, 1>;
    ensure_smem(fn, smem);
    int cap = 0;
    if (const char* e = std::getenv("LOVE_UPD_GRID")) cap = std::atoi(e);
    if (cap <= 0) {
        int dev = 0, sms = 0, per = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, smem), "update occupancy");
        cap = std::max(1, sms * per);
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nchunks, 256 / cg), cap));
}
template int update_grid<float>(int64_t, size_t, int);
template int update_grid<double>(int64_t, size_t, int);

// ---- ReplayThrottle (love_internal.h).  Per (thread, device): one mapped host int and a ring
// of kReplayWindow events, created once.
constexpr int kReplayWindow = 3;
ReplayThrottle::ReplayThrottle(int device) {
    struct Slot {
        int* h = nullptr;
        int* d = nullptr;
        cudaEvent_t ev[kReplayWindow] = {};
    };
    thread_local Slot slots[64];
    if (device < 0 || device >= 64) throw LoveError{LOVE_ERR_CUDA, "device index out of range"};
    Slot& sl = slots[device];
    if (sl.h == nullptr) {
        cuda_check(cudaHostAlloc((void**)&sl.h, 64, cudaHostAllocMapped), "cudaHostAlloc(done flag)");
        cuda_check(cudaHostGetDevicePointer((void**)&sl.d, sl.h, 0), "cudaHostGetDevicePointer");
        for (int i = 0; i < kReplayWindow; ++i)
            cuda_check(cudaEventCreateWithFlags(&sl.ev[i], cudaEventDisableTiming), "event create");
    }
    *(volatile int*)sl.h = 0;
    h = sl.h;
    d = sl.d;
    ev = sl.ev;
}

bool ReplayThrottle::admit(int i) {
    if (stopped()) return false;
    if (i >= kReplayWindow) {
        cuda_check(cudaEventSynchronize(ev[i % kReplayWindow]), "replay window");
        if (stopped()) return false;
    }
    return true;
}

void ReplayThrottle::launched(int i, cudaStream_t s) {
    cuda_check(cudaEventRecord(ev[i % kReplayWindow], s), "replay event");
}

// L2 residency of the Lanczos basis' first columns: both reorthogonalisation passes of every
// step read columns 0, 1, ..., so when Q~ is several times the L2 the first 48 MB of it are
// marked persisting for the build (stream access-policy window, inherited by the captured
// kernel nodes) and released afterwards.  Measured (same-box A/B, MB set aside): cfg2 (Q~
// 404 MB) 10.27 -> 10.17 ms at 48 / 64; cfg4 (808 MB) 29.91 -> 29.35 ms at 48, 31.05 at 72;
// cfg3 (202 MB) and cfg5 (80 MB, already L2-sized) slower.  LOVE_L2_PERSIST = MB (0: off).
struct L2Persist {
    cudaStream_t s = nullptr;
    bool on = false;
    size_t prev_limit = 0;                    // the device's set-aside before the build (restored)
    L2Persist(const Cache& c, cudaStream_t st) : s(st) {
        if (c.comm != nullptr || c.Q == nullptr) return;
        const size_t qbytes = c.vsize * (size_t)c.ldq * (size_t)(c.k_req + 1);
        const char* e = std::getenv("LOVE_L2_PERSIST");
        const double mb = e ? std::atof(e) : (qbytes >= (size_t(384) << 20) ? 48.0 : 0.0);
        if (!(mb > 0.0)) return;
        int dev = 0, maxp = 0, maxw = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        if (maxp <= 0 || maxw <= 0) return;
        const size_t persist = std::min<size_t>((size_t)(mb * 1048576.0), (size_t)maxp);
        const size_t window = std::min<size_t>({persist, (size_t)maxw, qbytes});
        if (cudaDeviceGetLimit(&prev_limit, cudaLimitPersistingL2CacheSize) != cudaSuccess) return;
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist) != cudaSuccess) return;
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.base_ptr = c.Q;
        v.accessPolicyWindow.num_bytes = window;
        v.accessPolicyWindow.hitRatio = 1.0f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        on = cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
        if (std::getenv("LOVE_L2_DEBUG"))
            std::fprintf(stderr, "[love l2] max persist %d MB, max window %d MB, window %.1f MB, on %d\n",
                         maxp >> 20, maxw >> 20, window / 1048576.0, (int)on);
    }
    ~L2Persist() {
        if (!on) return;
        cudaStreamAttrValue v = {};
        v.accessPolicyWindow.num_bytes = 0;
        cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev_limit);
    }
};

void* l2_persist_begin(const Cache& c, cudaStream_t s) {
    L2Persist* p = new L2Persist(c, s);
    if (!p->on) {
        delete p;
        return nullptr;
    }
    return p;
}
void l2_persist_end(void* h) { delete static_cast<L2Persist*>(h); }

void run_lanczos(Cache& c, cudaStream_t s) {
    if (c.precision == LOVE_FP64) lanczos_impl<double>(c, s);
    else lanczos_impl<float>(c, s);
}

void avgcol_probe(Cache& c, cudaStream_t s) {
    ProfScope ps(LOVE_PROF_SETUP, s);
    if (c.precision == LOVE_FP64) avgcol_impl<double>(c, s);
    else avgcol_impl<float>(c, s);
}

void mean_cache_eq4(Cache& c, cudaStream_t s) {
    ProfScope ps(LOVE_PROF_FINISH, s);
    if (c.precision == LOVE_FP64) eq4_impl<double>(c, s);
    else eq4_impl<float>(c, s);
}

void finish_cache(Cache& c, cudaStream_t s) {
    ProfScope ps(LOVE_PROF_FINISH, s);
    const int m = c.g.m_total;
    c.k_pad = (int)round_up(std::max(c.k_eff, 1), 4);
    c.Rc = dalloc(c, c.vsize * (size_t)m * c.k_pad, s);
    dim3 grid((unsigned)ceil_div(m, 32), (unsigned)ceil_div(c.k_pad, 32));
    dim3 block(32, 8);
    if (c.precision == LOVE_FP64)
        LOVE_LAUNCH(rc_transpose_kernel<double>, grid, block, 0, s, (const double*)c.Rc_col, m, c.k_eff, c.k_pad,
                    (double*)c.Rc);
    else
        LOVE_LAUNCH(rc_transpose_kernel<float>, grid, block, 0, s, (const double*)c.Rc_col, m, c.k_eff, c.k_pad,
                    (float*)c.Rc);
}

// fp64 row-major copy of the cache (m x k_pad) from the fp64 streamed Rc: fp32 caches answer
// covariances from it (love_predict_covar).  `out` holds m * k_pad doubles.
void launch_rc_rows64(const Cache& c, double* out, cudaStream_t s) {
    const int m = c.g.m_total;
    dim3 grid((unsigned)ceil_div(m, 32), (unsigned)ceil_div(c.k_pad, 32));
    dim3 block(32, 8);
    LOVE_LAUNCH(rc_transpose_kernel<double>, grid, block, 0, s, (const double*)c.Rc_col, m, c.k_eff, c.k_pad, out);
}

}  // namespace love
