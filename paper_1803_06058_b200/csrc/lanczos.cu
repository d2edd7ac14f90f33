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

#include "love_internal.h"

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

// ---- per-step scalar bookkeeping (one thread).  Finalises index i = j-1: alpha_i, the
// Cholesky row i of T, g_i, then beta_i, the breakdown test and the scale of q_j.
__global__ void lanczos_scalars_kernel(LanczosState st, int j, int k, double tol) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int* fl = st.flags;
    if (j == 0) {
        const double b2 = st.bnorm2[0];
        if (!(b2 > 0.0)) { fl[3] = 1; fl[0] = 1; fl[1] = 0; return; }
        st.qscale[0] = 1.0 / sqrt(b2);
        return;
    }
    if (fl[0]) return;
    const int i = j - 1;
    const double a = st.alpha_acc[i];
    st.alpha[i] = a;
    st.amax_bmax[0] = fmax(st.amax_bmax[0], fabs(a));
    const double lsub = i > 0 ? st.Ls[i - 1] : 0.0;
    const double piv = a - lsub * lsub;
    if (!(piv > 0.0)) { fl[2] = 1; fl[0] = 1; fl[1] = i; return; }
    const double ld = sqrt(piv);
    st.Ld[i] = ld;
    st.g[i] = (i == 0) ? 1.0 / ld : -lsub * st.g[i - 1] / ld;
    if (j == k) { fl[0] = 1; fl[1] = k; return; }
    const double b = sqrt(st.beta2_acc[i]);
    st.amax_bmax[1] = fmax(st.amax_bmax[1], b);
    if (!(b >= tol * (st.amax_bmax[0] + 2.0 * st.amax_bmax[1]))) { fl[0] = 1; fl[1] = j; return; }
    st.beta[i] = b;
    st.Ls[i] = b / ld;
    st.qscale[j] = 1.0 / b;
}

// Rc[:, i] = (z_i - L_{i,i-1} Rc[:, i-1]) / L_ii ;  a += ||b|| g_i Rc[:, i]    (fp64)
template <typename V>
__global__ void rc_update_kernel(LanczosState st, int i, int m, const V* __restrict__ z,
                                 double* __restrict__ Rc, double* __restrict__ a, int mean_y) {
    if (i >= st.flags[1] || st.flags[2] || st.flags[3]) return;
    const double ld = st.Ld[i];
    const double ls = i > 0 ? st.Ls[i - 1] : 0.0;
    const double ag = sqrt(st.bnorm2[0]) * st.g[i];
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
        const double prev = i > 0 ? Rc[(int64_t)(i - 1) * m + p] : 0.0;
        const double v = ((double)z[p] - ls * prev) / ld;
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

// ---- reorthogonalisation dots: c[i] += q_i^T src over this CTA's rows, i = 0..j.
// One row tile per CTA (tiles sized so the grid is ~2 CTAs per SM); warps own columns and
// stream Q~[tile, col] with 16-byte loads against the tile of src staged in shared memory.
template <typename V>
__global__ void __launch_bounds__(256) reorth_dots_kernel(const V* __restrict__ Q, int64_t ldq,
                                                          int64_t tile_rows, int j,
                                                          const V* __restrict__ r, int from_r,
                                                          LanczosState st, double* __restrict__ c_out) {
    constexpr int W = VecT<V>::W;
    constexpr int U = 4;
    extern __shared__ __align__(16) double smd[];
    if (st.flags[0]) return;
    const int ncols = j + 1;
    double* csum = smd;                                   // [ncols]
    V* src = reinterpret_cast<V*>(smd + round_up(ncols, 2));   // [tile_rows]
    const int64_t row0 = (int64_t)blockIdx.x * tile_rows;
    const int64_t rows = min(tile_rows, ldq - row0);
    if (rows <= 0) return;
    for (int i = threadIdx.x; i < ncols; i += blockDim.x) csum[i] = 0.0;
    const double sj = st.qscale[j];
    const double aj = st.alpha_acc[j] * sj;
    const double bj1 = j > 0 ? st.beta[j - 1] * st.qscale[j - 1] : 0.0;
    const int nchunk = (int)(rows / W);
    for (int q = threadIdx.x; q < nchunk; q += blockDim.x) {
        double v[W];
        load_src<V>(Q, ldq, r, from_r, j, aj, bj1, row0 + (int64_t)q * W, v);
#pragma unroll
        for (int e = 0; e < W; ++e) src[q * W + e] = (V)v[e];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int col = wid; col < ncols; col += nw) {
        const V* qc = Q + (int64_t)col * ldq + row0;
        V part = V(0);
        for (int q0 = lane; q0 < nchunk; q0 += 32 * U) {
            V a[U][W], b[U][W];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = q0 + 32 * u;
                if (q < nchunk) {
                    vload<V>(qc + q * W, a[u]);
                    vload<V>(src + q * W, b[u]);
                } else {
#pragma unroll
                    for (int e = 0; e < W; ++e) a[u][e] = b[u][e] = V(0);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int e = 0; e < W; ++e) part += a[u][e] * b[u][e];
        }
        const double dp = warp_sum((double)part);
        if (lane == 0) csum[col] = dp;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ncols; i += blockDim.x) atomicAdd(&c_out[i], csum[i] * st.qscale[i]);
}

// ---- reorthogonalisation update: Q~[:, j+1] = src - sum_i c_i q_i ; beta2 += ||.||^2
template <typename V>
__global__ void __launch_bounds__(256) reorth_update_kernel(V* __restrict__ Q, int64_t ldq, int64_t n, int j,
                                                            const V* __restrict__ r, int from_r,
                                                            LanczosState st, const double* __restrict__ c_in,
                                                            double* __restrict__ beta2_out) {
    constexpr int W = VecT<V>::W;
    extern __shared__ double cf[];             // [j+1] coefficient of Q~[:, i]
    __shared__ double red[32];
    if (st.flags[0]) return;
    const int ncols = j + 1;
    for (int i = threadIdx.x; i < ncols; i += blockDim.x) cf[i] = c_in[i] * st.qscale[i];
    __syncthreads();
    const double sj = st.qscale[j];
    const double aj = st.alpha_acc[j] * sj;
    const double bj1 = j > 0 ? st.beta[j - 1] * st.qscale[j - 1] : 0.0;
    double b2 = 0.0;
    const int64_t nchunks = ldq / W;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nchunks;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = q * W;
        double v[W];
        load_src<V>(Q, ldq, r, from_r, j, aj, bj1, p, v);
        V acc[W];
#pragma unroll
        for (int e = 0; e < W; ++e) acc[e] = V(0);
#pragma unroll 4
        for (int i = 0; i < ncols; ++i) {
            V a[W];
            vload<V>(Q + (int64_t)i * ldq + p, a);
            const V ci = (V)cf[i];
#pragma unroll
            for (int e = 0; e < W; ++e) acc[e] += ci * a[e];
        }
        V o[W];
#pragma unroll
        for (int e = 0; e < W; ++e) {
            o[e] = (p + e < n) ? (V)(v[e] - (double)acc[e]) : V(0);
            b2 += (double)o[e] * (double)o[e];
        }
        vstore<V>(Q + (int64_t)(j + 1) * ldq + p, o);
    }
    if (beta2_out != nullptr) {
        b2 = block_sum(b2, red);
        if (threadIdx.x == 0) atomicAdd(beta2_out, b2);
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

// rows per dots tile: ~2 CTAs per SM, a multiple of 32 vector chunks
template <typename V>
int64_t reorth_tile_rows(int64_t ldq) {
    const int64_t quantum = 32 * VecT<V>::W;
    return std::max<int64_t>(quantum, round_up(ceil_div(ldq, 148 * 2), quantum));
}

template <typename V>
void lanczos_impl(Cache& c, cudaStream_t s) {
    const int k = c.k_req;
    const int m = c.g.m_total;
    const int64_t ldq = c.ldq;
    V* Q = (V*)c.Q;
    V* r = (V*)c.r;
    V* u = (V*)c.u;
    double* Rcc = (double*)c.Rc_col;
    double* a = (double*)c.a;
    const LanczosState& st = c.st;
    const int P = c.reorth_passes;
    const int mean_y = c.probe == LOVE_PROBE_Y;
    const int gm = (int)std::min<int64_t>(ceil_div(m, 256), 148 * 8);
    const int64_t tile_rows = reorth_tile_rows<V>(ldq);
    const int gr = (int)ceil_div(ldq, tile_rows);
    const int gu = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ldq / VecT<V>::W, 256), 148 * 8));

    LOVE_LAUNCH(norm2_kernel<V>, (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(c.n, 256), 148 * 4)), 256,
                0, s, Q, c.n, st.bnorm2);
    if (c.world > 1) allreduce_sum(c, st.bnorm2, 1, true, s);
    for (int j = 0; j < k; ++j) {
        LOVE_LAUNCH(lanczos_scalars_kernel, 1, 32, 0, s, st, j, k, c.tol);
        if (j > 0)
            LOVE_LAUNCH(rc_update_kernel<V>, gm, 256, 0, s, st, j - 1, m, (const V*)c.z[(j - 1) & 1], Rcc, a,
                        mean_y);
        const V* qj = Q + (int64_t)j * ldq;
        V* zj = (V*)c.z[j & 1];
        launch_scatter<V>(c, qj, st.qscale + j, u, s);
        if (c.world > 1) allreduce_sum(c, u, m, sizeof(V) == 8, s);
        launch_kuu<V>(c, u, zj, s);
        launch_gather<V>(c, zj, qj, st.qscale + j, r, st.alpha_acc + j, s);
        if (c.world > 1) allreduce_sum(c, st.alpha_acc + j, 1, true, s);
        if (j == k - 1) break;
        for (int pass = 0; pass < P; ++pass) {
            double* cacc = st.c_acc + ((int64_t)(pass & 1) * k + j) * (k + 1);
            if (pass >= 2) cuda_check(cudaMemsetAsync(cacc, 0, sizeof(double) * (k + 1), s), "c zero");
            const int from_r = pass == 0;
            const size_t smd = sizeof(double) * round_up(j + 1, 2) + sizeof(V) * tile_rows;
            LOVE_LAUNCH(reorth_dots_kernel<V>, gr, 256, smd, s, Q, ldq, tile_rows, j, r, from_r, st, cacc);
            if (c.world > 1) allreduce_sum(c, cacc, j + 1, true, s);
            LOVE_LAUNCH(reorth_update_kernel<V>, gu, 256, sizeof(double) * (j + 1), s, Q, ldq, c.n, j, r, from_r,
                        st, cacc, pass == P - 1 ? st.beta2_acc + j : nullptr);
        }
        if (c.world > 1) allreduce_sum(c, st.beta2_acc + j, 1, true, s);
    }
    LOVE_LAUNCH(lanczos_scalars_kernel, 1, 32, 0, s, st, k, k, c.tol);
    LOVE_LAUNCH(rc_update_kernel<V>, gm, 256, 0, s, st, k - 1, m, (const V*)c.z[(k - 1) & 1], Rcc, a, mean_y);
}

}  // namespace

void run_lanczos(Cache& c, cudaStream_t s) {
    if (c.precision == LOVE_FP64) lanczos_impl<double>(c, s);
    else lanczos_impl<float>(c, s);
}

void finish_cache(Cache& c, cudaStream_t s) {
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

}  // namespace love
