// query.cu -- O(k) predictive (co)variance and mean queries (Eq. 10; Alg. 1
// P:401-403; Eq. 6).
//
// One warp per query.  Interpolation (cell, Keys weights) and the prior are computed in
// fp64 (reading A21: the cancellation prior - ||Rc^T w||^2 needs fp64 weights); lanes own
// 16-byte chunks of the k-vector r = sum_l w_l Rc[node_l, :] and accumulate in fp64.  For
// d = 1 the 4 stencil rows of Rc are contiguous (4 * k_pad values), for d = 3 they are 16
// runs of 4 rows.
#include <cuda_runtime.h>

#include <cuda_pipeline.h>

#include <cmath>
#include <cstdlib>

#include "love_internal.h"
#include "ski_device.cuh"
#include "tma.cuh"

#ifndef LOVE_SORTED3_TMA
#define LOVE_SORTED3_TMA 1
#endif

#ifndef LOVE_SORTED3_BALANCE
#define LOVE_SORTED3_BALANCE 1
#endif
constexpr bool kSorted3Balance = LOVE_SORTED3_BALANCE;   // d = 3 lane mode: remainder groups split k

#ifndef LOVE_SORTED3_HOIST
#define LOVE_SORTED3_HOIST 1
#endif
constexpr bool kSorted3Hoist = LOVE_SORTED3_HOIST;       // lane-mode weights packed once per query

#ifndef LOVE_PAIRED_Q3
#define LOVE_PAIRED_Q3 1
#endif

namespace love {

namespace {

template <typename V> struct QV;
template <> struct QV<float> { using T = float4; static constexpr int W = 4; };
template <> struct QV<double> { using T = double2; static constexpr int W = 2; };

struct Stencil {
    int base;            // flat node index of the stencil origin (cell - 1 per dim)
    int j[3];            // cell per dim
    double w[3][4];      // Keys weights per dim
    bool ok;
};

template <int D>
__device__ __forceinline__ Stencil make_stencil(const GridDev& g, const double* x) {
    Stencil s;
    s.ok = true;
    s.base = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        s.j[d] = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) s.w[d][e] = 0.0;
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const double sc = (x[d] - g.lo[d]) / g.h[d];
        const double jf = floor(sc);
        const bool bad = !(jf >= 1.0 && jf <= (double)(g.m[d] - 3));   // reading A4
        s.ok = s.ok && !bad;
        const int j = bad ? 1 : (int)jf;
        s.j[d] = j;
        keys4<double>(bad ? 0.0 : sc - jf, s.w[d]);
        s.base += (j - 1) * g.stride[d];
    }
    return s;
}

// SKI prior w_a^T K_UU w_b = s^2 prod_d sum_{a,b} w_a[d][a] w_b[d][b] c_d[|(ja+a)-(jb+b)|]
// (Eq. 12 first term; K_UU entries P:187)
template <int D>
__device__ __forceinline__ double prior_ski(const GridDev& g, const double* cols64, double s2,
                                            const Stencil& A, const Stencil& B) {
    double p = s2;
    int off = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                acc += A.w[d][a] * B.w[d][b] * cols64[off + abs((A.j[d] + a) - (B.j[d] + b))];
        p *= acc;
        off += g.m[d];
    }
    return p;
}

// w[a] for a runtime a without dynamic register indexing (which would go to local memory)
__device__ __forceinline__ double pick4(const double w[4], int a) {
    return a == 0 ? w[0] : a == 1 ? w[1] : a == 2 ? w[2] : w[3];
}

// acc[e] = sum over the 4^d stencil rows l of w_l * Rc[node_l, ch*W + e]   (fp64)
template <typename V, int D>
__device__ __forceinline__ void stencil_rows(const GridDev& g, const Stencil& S, const V* __restrict__ Rc,
                                             int k_pad, int ch, double acc[QV<V>::W]) {
    constexpr int W = QV<V>::W;
    using VT = typename QV<V>::T;
#pragma unroll
    for (int e = 0; e < W; ++e) acc[e] = 0.0;
    constexpr int UA = D >= 2 ? 1 : 4;        // bound registers for the 16- and 64-row stencils
#pragma unroll UA
    for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < (D > 1 ? 4 : 1); ++b) {
#pragma unroll
            for (int cc = 0; cc < (D > 2 ? 4 : 1); ++cc) {
                int node = S.base;
                double w = pick4(S.w[0], a);
                if (D == 1) node += a;
                if (D == 2) { node += a * g.stride[0] + b; w *= S.w[1][b]; }
                if (D == 3) {
                    node += a * g.stride[0] + b * g.stride[1] + cc;
                    w *= S.w[1][b] * S.w[2][cc];
                }
                const VT v = __ldg(reinterpret_cast<const VT*>(Rc + (int64_t)node * k_pad + ch * W));
                if constexpr (W == 4) {
                    acc[0] += w * (double)v.x; acc[1] += w * (double)v.y;
                    acc[2] += w * (double)v.z; acc[3] += w * (double)v.w;
                } else {
                    acc[0] += w * (double)v.x; acc[1] += w * (double)v.y;
                }
            }
        }
    }
}

// first 4 entries of each Toeplitz column: all a variance query's prior needs
struct C4 {
    double c[3][4];
};

// G lanes cooperate on one query (32/G queries per warp in flight); lane gl owns the
// 16-byte chunks gl, gl+G, ... of the k-vector, for all 4^d stencil rows.
template <typename V, int D, int G>
__global__ void __launch_bounds__(256) predict_kernel(GridDev g, const double* __restrict__ cols64, C4 c4,
                                                      double s2, double l0, double l1, double l2, int prior_mode,
                                                      const V* __restrict__ Rc, int k_pad,
                                                      const double* __restrict__ amean,
                                                      const double* __restrict__ Xa,
                                                      const double* __restrict__ Xb, int64_t t,
                                                      V* __restrict__ out, V* __restrict__ mean_out,
                                                      unsigned long long* __restrict__ counters) {
    constexpr int W = QV<V>::W;
    constexpr int QPW = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nchunks = k_pad / W;
    const bool covar = Xb != nullptr;
    for (int64_t base = warp * QPW; base < t; base += nwarps * QPW) {
        const int64_t qi = base + sub;
        const bool active = qi < t;
        const int64_t qq = active ? qi : base;
        const Stencil A = make_stencil<D>(g, Xa + qq * D);
        const Stencil B = covar ? make_stencil<D>(g, Xb + qq * D) : A;
        const bool ok = active && A.ok && B.ok;
        double dot = 0.0;
        if (ok) {
            for (int ch = gl; ch < nchunks; ch += G) {
                double ra[W], rb[W];
                stencil_rows<V, D>(g, A, Rc, k_pad, ch, ra);
                if (covar) stencil_rows<V, D>(g, B, Rc, k_pad, ch, rb);
                else
#pragma unroll
                    for (int e = 0; e < W; ++e) rb[e] = ra[e];
#pragma unroll
                for (int e = 0; e < W; ++e) dot += ra[e] * rb[e];
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (gl != 0 || !active) continue;
        if (!ok) {
            out[qi] = (V)NAN;
            if (mean_out) mean_out[qi] = (V)NAN;
            atomicAdd(&counters[1], 1ull);
            continue;
        }
        double prior;
        if (prior_mode == LOVE_PRIOR_EXACT) {
            const double ls[3] = {l0, l1, l2};
            double r2 = 0.0;
            for (int d = 0; d < D; ++d) {
                const double df = Xa[qi * D + d] - (covar ? Xb[qi * D + d] : Xa[qi * D + d]);
                r2 += df * df / (ls[d] * ls[d]);
            }
            prior = s2 * exp(-0.5 * r2);
        } else if (!covar) {
            // w^T K_UU w with the Kronecker structure: s^2 prod_d sum_ab w_a w_b c_d[|a-b|]
            prior = s2;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                double acc = 0.0;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc += A.w[d][a] * A.w[d][b] * c4.c[d][a > b ? a - b : b - a];
                prior *= acc;
            }
        } else {
            prior = prior_ski<D>(g, cols64, s2, A, B);
        }
        const double v = prior - dot;
        out[qi] = (V)v;
        if (!covar && v < 0.0) atomicAdd(&counters[0], 1ull);
        if (mean_out) {
            double mu = 0.0;
#pragma unroll 1
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < (D > 1 ? 4 : 1); ++b)
                    for (int cc = 0; cc < (D > 2 ? 4 : 1); ++cc) {
                        int node = A.base;
                        double w = pick4(A.w[0], a);
                        if (D == 1) node += a;
                        if (D == 2) { node += a * g.stride[0] + b; w *= A.w[1][b]; }
                        if (D == 3) {
                            node += a * g.stride[0] + b * g.stride[1] + cc;
                            w *= A.w[1][b] * A.w[2][cc];
                        }
                        mu += w * amean[node];
                    }
            mean_out[qi] = (V)mu;
        }
    }
}

// ---- per-cell variance blocks (SURVEY 8(f) NEXT #3b, d <= 2).  For a cell c with stencil
// nodes S_c (4^d of them), B_c = K_UU|S_c - (Rc Rc^T)|S_c in fp64, stored packed upper
// triangular (pairs a <= b in row-major order).  Eq. 10 with the SKI prior is then
//   var(x*) = w*^T K_UU w* - ||Rc^T w*||^2 = w*^T B_c w*   for x* in cell c.
// Rc is the fp64 column-major streamed cache (m x k_eff).
__host__ __device__ constexpr int blk_size(int D) { return D == 1 ? 10 : 136; }

__global__ void __launch_bounds__(256) var_blocks1_kernel(int m, int k_eff, const double* __restrict__ Rc,
                                                          const double* __restrict__ c0, double s2,
                                                          double* __restrict__ blk) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m) return;
    double* out = blk + (int64_t)c * 10;
    if (c < 1 || c > m - 3) {
#pragma unroll
        for (int p = 0; p < 10; ++p) out[p] = 0.0;
        return;
    }
    double acc[10];
#pragma unroll
    for (int p = 0; p < 10; ++p) acc[p] = 0.0;
    for (int i = 0; i < k_eff; ++i) {
        const double* col = Rc + (int64_t)i * m + (c - 1);
        const double r0 = col[0], r1 = col[1], r2 = col[2], r3 = col[3];
        acc[0] += r0 * r0; acc[1] += r0 * r1; acc[2] += r0 * r2; acc[3] += r0 * r3;
        acc[4] += r1 * r1; acc[5] += r1 * r2; acc[6] += r1 * r3;
        acc[7] += r2 * r2; acc[8] += r2 * r3;
        acc[9] += r3 * r3;
    }
    int p = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = a; b < 4; ++b, ++p) out[p] = s2 * c0[b - a] - acc[p];
}

// d = 2: one warp per cell; lanes 0..15 load the 16 node values of Rc column i, every lane
// owns pairs p = lane, lane + 32, ... of the 136 and pulls the two values by shuffles.
__global__ void __launch_bounds__(256) var_blocks2_kernel(GridDev g, int k_eff, const double* __restrict__ Rc,
                                                          const double* __restrict__ cols, double s2,
                                                          double* __restrict__ blk) {
    const int lane = threadIdx.x & 31;
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int m = g.m_total;
    if (c >= m) return;
    const int ci = c / g.m[1], cj = c - ci * g.m[1];
    double* out = blk + (int64_t)c * 136;
    const bool ok = ci >= 1 && ci <= g.m[0] - 3 && cj >= 1 && cj <= g.m[1] - 3;
    int pa[5], pb[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {           // pair index -> (a, b), a <= b, row-major over a
        int p = lane + 32 * t, a = 0;
        while (p >= 16 - a && a < 16) { p -= 16 - a; ++a; }
        pa[t] = a;
        pb[t] = a + p;
    }
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const int node = ok ? (ci - 1 + (lane >> 2)) * g.m[1] + (cj - 1 + (lane & 3)) : 0;
    if (ok) {
        for (int i = 0; i < k_eff; ++i) {
            const double v = lane < 16 ? Rc[(int64_t)i * m + node] : 0.0;
#pragma unroll
            for (int t = 0; t < 5; ++t) {
                const double va = __shfl_sync(0xffffffffu, v, pa[t] & 15);
                const double vb = __shfl_sync(0xffffffffu, v, pb[t] & 15);
                acc[t] += va * vb;
            }
        }
    }
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int p = lane + 32 * t;
        if (p >= 136) continue;
        const int a = pa[t], b = pb[t];
        const double kuu = s2 * cols[abs((a >> 2) - (b >> 2))] * cols[g.m[0] + abs((a & 3) - (b & 3))];
        out[p] = ok ? kuu - acc[t] : 0.0;
    }
}

// d = 2 blocks from node-pair products.  B_c[a][b] (a <= b, row-major over the 4x4 stencil
// of cell c) only depends on the node pair (n_a, n_b) = (n_a, n_a + off) with off = (di, dj)
// in the half neighbourhood H = {di = 0, 0 <= dj <= 3} u {1 <= di <= 3, |dj| <= 3} (25
// offsets): B_c[a][b] = K_UU[n_a][n_b] - P[off][n_a], P[off][n] = sum_i Rc[n, i] Rc[n + off, i].
// A node pair is shared by up to 16 cells, so the products are formed once per pair (25 m k
// FMAs instead of 136 m k), tile by tile from shared memory; the assembly is a gather.
constexpr int kPairOffs = 25;
__host__ __device__ __forceinline__ void pair_off(int o, int& di, int& dj) {
    if (o < 4) { di = 0; dj = o; }
    else { di = 1 + (o - 4) / 7; dj = (o - 4) % 7 - 3; }
}
__host__ __device__ __forceinline__ int pair_index(int di, int dj) {   // inverse of pair_off
    return di == 0 ? dj : 4 + (di - 1) * 7 + (dj + 3);
}
constexpr int kPTI = 8, kPTJ = 32, kPB = 8;   // node tile (rows x cols) and Rc columns per stage

__global__ void __launch_bounds__(kPTI * kPTJ) pair_products2_kernel(GridDev g, int k_eff,
                                                                      const double* __restrict__ Rc,
                                                                      double* __restrict__ P) {
    constexpr int HI = kPTI + 3, HJ = kPTJ + 6;         // halo: +3 rows, -3..+3 columns
    __shared__ double tile[kPB][HI][HJ];
    const int m = g.m_total, m0 = g.m[0], m1 = g.m[1];
    const int ti = threadIdx.x / kPTJ, tj = threadIdx.x % kPTJ;
    const int i0 = blockIdx.y * kPTI, j0 = blockIdx.x * kPTJ;
    const int ni = i0 + ti, nj = j0 + tj;
    double acc[kPairOffs];
#pragma unroll
    for (int o = 0; o < kPairOffs; ++o) acc[o] = 0.0;
    for (int c0 = 0; c0 < k_eff; c0 += kPB) {
        for (int e = threadIdx.x; e < kPB * HI * HJ; e += blockDim.x) {
            const int b = e / (HI * HJ), r = (e / HJ) % HI, q = e % HJ;
            const int gi = i0 + r, gj = j0 + q - 3, col = c0 + b;
            tile[b][r][q] = (col < k_eff && gi < m0 && gj >= 0 && gj < m1) ? Rc[(int64_t)col * m + gi * m1 + gj] : 0.0;
        }
        __syncthreads();
#pragma unroll 2
        for (int b = 0; b < kPB; ++b) {
            const double x = tile[b][ti][tj + 3];
#pragma unroll
            for (int o = 0; o < kPairOffs; ++o) {
                int di, dj;
                pair_off(o, di, dj);
                acc[o] += x * tile[b][ti + di][tj + 3 + dj];
            }
        }
        __syncthreads();
    }
    if (ni < m0 && nj < m1) {
#pragma unroll
        for (int o = 0; o < kPairOffs; ++o) P[(int64_t)o * m + ni * m1 + nj] = acc[o];
    }
}

// thread per block entry: B_c[p] = s^2 c0[|di|] c1[|dj|] - P[off][n_a] (0 for cells whose
// stencil leaves the grid)
__global__ void __launch_bounds__(256) assemble_blocks2_kernel(GridDev g, const double* __restrict__ P,
                                                               const double* __restrict__ cols, double s2,
                                                               double* __restrict__ blk) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int m = g.m_total;
    if (e >= (int64_t)m * 136) return;
    const int c = (int)(e / 136), p0 = (int)(e - (int64_t)c * 136);
    const int ci = c / g.m[1], cj = c - ci * g.m[1];
    const bool ok = ci >= 1 && ci <= g.m[0] - 3 && cj >= 1 && cj <= g.m[1] - 3;
    if (!ok) {
        blk[e] = 0.0;
        return;
    }
    int p = p0, a = 0;
    while (p >= 16 - a) { p -= 16 - a; ++a; }
    const int b = a + p;
    const int di = (b >> 2) - (a >> 2), dj = (b & 3) - (a & 3);
    const int na = (ci - 1 + (a >> 2)) * g.m[1] + (cj - 1 + (a & 3));
    const double kuu = s2 * cols[di] * cols[g.m[0] + (dj < 0 ? -dj : dj)];
    blk[e] = kuu - P[(int64_t)pair_index(di, dj) * m + na];
}

// variance (and mean) of one query from its cell block (fp64)
template <typename V, int D>
__device__ __forceinline__ void block_query(const GridDev& g, const C4& c4, double s2, int prior_mode,
                                            const double* __restrict__ blk, const double* __restrict__ amean,
                                            const Stencil& A, int64_t qi, V* __restrict__ out,
                                            V* __restrict__ mean_out, unsigned long long* __restrict__ counters) {
    if (!A.ok) {
        out[qi] = (V)NAN;
        if (mean_out) mean_out[qi] = (V)NAN;
        atomicAdd(&counters[1], 1ull);
        return;
    }
    constexpr int S = D == 1 ? 4 : 16;
    double w[S];
#pragma unroll
    for (int a = 0; a < S; ++a) w[a] = D == 1 ? A.w[0][a] : A.w[0][a >> 2] * A.w[1][a & 3];
    const int cell = D == 1 ? A.j[0] : A.j[0] * g.m[1] + A.j[1];
    const double* __restrict__ B = blk + (int64_t)cell * blk_size(D);
    double v = 0.0;
    int p = 0;
    if constexpr (D == 1) {                      // the 80-byte block as five 16-byte loads
        double bb[10];
#pragma unroll
        for (int h = 0; h < 5; ++h) {
            const double2 x = __ldg(reinterpret_cast<const double2*>(B) + h);
            bb[2 * h] = x.x;
            bb[2 * h + 1] = x.y;
        }
#pragma unroll
        for (int a = 0; a < S; ++a) {
            double row = 0.5 * w[a] * bb[p++];
#pragma unroll
            for (int b = a + 1; b < S; ++b) row += w[b] * bb[p++];
            v += 2.0 * w[a] * row;
        }
    } else {
#pragma unroll
    for (int a = 0; a < S; ++a) {
        double row = 0.5 * w[a] * __ldg(B + p++);
#pragma unroll
        for (int b = a + 1; b < S; ++b) row += w[b] * __ldg(B + p++);
        v += 2.0 * w[a] * row;
    }
    }
    if (prior_mode == LOVE_PRIOR_EXACT) {
        // k(x*, x*) - w^T K_UU w + w^T B w   (the exact prior of Eq. 10)
        double pr = s2;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc += A.w[d][a] * A.w[d][b] * c4.c[d][a > b ? a - b : b - a];
            pr *= acc;
        }
        v += s2 - pr;
    }
    out[qi] = (V)v;
    if (v < 0.0) atomicAdd(&counters[0], 1ull);
    if (mean_out) {
        double mu = 0.0;
#pragma unroll
        for (int a = 0; a < S; ++a) {
            const int node = D == 1 ? A.base + a : A.base + (a >> 2) * g.stride[0] + (a & 3);
            mu += w[a] * __ldg(amean + node);
        }
        mean_out[qi] = (V)mu;
    }
}

// QPT queries per thread (queries base + u * blockDim + tid): their stencils are computed
// before any block is read, so each thread has QPT independent dependent-load chains in flight
template <typename V, int D, int QPT>
__global__ void __launch_bounds__(256) predict_block_kernel(GridDev g, C4 c4, double s2, int prior_mode,
                                                            const double* __restrict__ blk,
                                                            const double* __restrict__ amean,
                                                            const double* __restrict__ Xs, int64_t t,
                                                            V* __restrict__ out, V* __restrict__ mean_out,
                                                            unsigned long long* __restrict__ counters) {
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * QPT + threadIdx.x;
    Stencil A[QPT];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        const int64_t qi = base + (int64_t)u * blockDim.x;
        A[u] = make_stencil<D>(g, Xs + (qi < t ? qi : 0) * D);
    }
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        const int64_t qi = base + (int64_t)u * blockDim.x;
        if (qi < t) block_query<V, D>(g, c4, s2, prior_mode, blk, amean, A[u], qi, out, mean_out, counters);
    }
}

// G lanes per query (d = 1: G = 2, d = 2: G = 8): the same w^T B_c w as block_query, with the
// block's packed entries p read by lane p % G (each group's loads are contiguous: 64 B per load
// instruction per query instead of one 8-byte load per entry and thread) and the 4^d fp64
// stencil weights shared through shared memory; the partial sums meet by shuffles.
template <typename V, int D, int G>
__global__ void __launch_bounds__(256) predict_block_coop_kernel(GridDev g, C4 c4, double s2, int prior_mode,
                                                                 const double* __restrict__ blk,
                                                                 const double* __restrict__ amean,
                                                                 const double* __restrict__ Xs, int64_t t,
                                                                 V* __restrict__ out, V* __restrict__ mean_out,
                                                                 unsigned long long* __restrict__ counters) {
    constexpr int S = D == 1 ? 4 : 16;
    constexpr int NB = S * (S + 1) / 2;            // 10 / 136 packed upper-triangular entries
    constexpr int QPB = 256 / G;                   // queries per CTA
    __shared__ unsigned char pa[NB], pb[NB];
    __shared__ double ws[QPB][S];
    for (int p = threadIdx.x; p < NB; p += blockDim.x) {
        int a = 0, r = p;
        while (r >= S - a) { r -= S - a; ++a; }
        pa[p] = (unsigned char)a;
        pb[p] = (unsigned char)(a + r);
    }
    const int gl = threadIdx.x % G, ql = threadIdx.x / G;
    const int64_t qi = (int64_t)blockIdx.x * QPB + ql;
    const bool live = qi < t;
    const Stencil A = make_stencil<D>(g, Xs + (live ? qi : 0) * D);
    for (int a = gl; a < S; a += G) ws[ql][a] = D == 1 ? pick4(A.w[0], a) : pick4(A.w[0], a >> 2) * pick4(A.w[1], a & 3);
    __syncthreads();
    const bool ok = live && A.ok;
    double v = 0.0, mu = 0.0;
    if (ok) {
        const int cell = D == 1 ? A.j[0] : A.j[0] * g.m[1] + A.j[1];
        const double* __restrict__ B = blk + (int64_t)cell * blk_size(D);
#pragma unroll
        for (int p = gl; p < NB; p += G) {
            const int a = pa[p], b = pb[p];
            const double wab = ws[ql][a] * ws[ql][b];
            v += (a == b ? wab : 2.0 * wab) * __ldg(B + p);
        }
        if (mean_out) {
            for (int a = gl; a < S; a += G) {
                const int node = D == 1 ? A.base + a : A.base + (a >> 2) * g.stride[0] + (a & 3);
                mu += ws[ql][a] * __ldg(amean + node);
            }
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        mu += __shfl_xor_sync(0xffffffffu, mu, o);
    }
    if (gl != 0 || !live) return;
    if (!A.ok) {
        out[qi] = (V)NAN;
        if (mean_out) mean_out[qi] = (V)NAN;
        atomicAdd(&counters[1], 1ull);
        return;
    }
    if (prior_mode == LOVE_PRIOR_EXACT) {          // k(x*, x*) - w^T K_UU w + w^T B w  (Eq. 10)
        double pr = s2;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc += A.w[d][a] * A.w[d][b] * c4.c[d][a > b ? a - b : b - a];
            pr *= acc;
        }
        v += s2 - pr;
    }
    out[qi] = (V)v;
    if (v < 0.0) atomicAdd(&counters[0], 1ull);
    if (mean_out) mean_out[qi] = (V)mu;
}

}  // namespace

// ---- d = 3 variance queries grouped by cell (SURVEY 8(f) NEXT #3a): the queries are
// counting-sorted by cell, a CTA stages the 64 stencil rows of Rc of one cell in shared
// memory once and every query of that cell reads them from there.
__global__ void query_cell3_kernel(GridDev g, const double* __restrict__ Xs, int64_t t, int* __restrict__ key) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < t; q += (int64_t)gridDim.x * blockDim.x) {
        int cell = 0;
        bool ok = true;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double jf = floor((Xs[q * 3 + d] - g.lo[d]) / g.h[d]);
            ok = ok && jf >= 1.0 && jf <= (double)(g.m[d] - 3);       // reading A4
            cell += (ok ? (int)jf : 0) * g.stride[d];
        }
        key[q] = ok ? cell : g.m_total;
    }
}

// variance (and mean) of one d = 3 query from its stencil, the reduced norm and the mean sum
template <typename V>
__device__ __forceinline__ void finish_sorted3(const Stencil& A, const C4& c4, double s2, int prior_mode, double dot,
                                               double mu, int q, V* __restrict__ out, V* __restrict__ mean_out,
                                               unsigned long long* __restrict__ counters) {
    double prior = s2;
    if (prior_mode != LOVE_PRIOR_EXACT) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc += A.w[d][a] * A.w[d][b] * c4.c[d][a > b ? a - b : b - a];
            prior *= acc;
        }
    }
    const double v = prior - dot;
    out[q] = (V)v;
    if (v < 0.0) atomicAdd(&counters[0], 1ull);
    if (mean_out) mean_out[q] = (V)mu;
}

// r = sum_a w0_a sum_b w1_b sum_c w2_c Rc[row(a,b,c)] on W consecutive k of the staged rows,
// innermost first; the 16-term (b, c) sums in the storage type V (fp32 rows in LOVE_FP32: a
// few ulp of fp32 on top of what the fp32 storage of Rc already carries, without converting
// every row element to fp64); the a-sum is fp64; returns sum_e r_e^2
template <typename V>
__device__ __forceinline__ double sorted3_chunk(const Stencil& A, const V* rows, int k_pad, int ch) {
    constexpr int W = QV<V>::W;
    using VT = typename QV<V>::T;
#if LOVE_PAIRED_Q3
    if constexpr (W == 4) {
        // fp32: the four k values as two FFMA2 pairs, the weights broadcast (same FMA per k)
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            f32x2 ra01 = 0ull, ra23 = 0ull;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                f32x2 rb01 = 0ull, rb23 = 0ull;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const float4 v = *reinterpret_cast<const float4*>(rows + (a * 16 + b * 4 + cc) * k_pad + ch * 4);
                    const float w = (float)A.w[2][cc];
                    const f32x2 ww = pk2(w, w);
                    rb01 = fma2(ww, pk2(v.x, v.y), rb01);
                    rb23 = fma2(ww, pk2(v.z, v.w), rb23);
                }
                const float w1b = (float)A.w[1][b];
                const f32x2 w1 = pk2(w1b, w1b);
                ra01 = fma2(w1, rb01, ra01);
                ra23 = fma2(w1, rb23, ra23);
            }
            acc[0] += A.w[0][a] * (double)lo2(ra01);
            acc[1] += A.w[0][a] * (double)hi2(ra01);
            acc[2] += A.w[0][a] * (double)lo2(ra23);
            acc[3] += A.w[0][a] * (double)hi2(ra23);
        }
        double dot = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) dot += acc[e] * acc[e];
        return dot;
    }
#endif
    double acc[W];
#pragma unroll
    for (int e = 0; e < W; ++e) acc[e] = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        V ra[W];
#pragma unroll
        for (int e = 0; e < W; ++e) ra[e] = V(0);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            V rb[W];
#pragma unroll
            for (int e = 0; e < W; ++e) rb[e] = V(0);
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const VT v = *reinterpret_cast<const VT*>(rows + (a * 16 + b * 4 + cc) * k_pad + ch * W);
                const V w = (V)A.w[2][cc];
                if constexpr (W == 4) {
                    rb[0] += w * v.x; rb[1] += w * v.y; rb[2] += w * v.z; rb[3] += w * v.w;
                } else {
                    rb[0] += w * v.x; rb[1] += w * v.y;
                }
            }
#pragma unroll
            for (int e = 0; e < W; ++e) ra[e] += (V)A.w[1][b] * rb[e];
        }
#pragma unroll
        for (int e = 0; e < W; ++e) acc[e] += A.w[0][a] * (double)ra[e];
    }
    double dot = 0.0;
#pragma unroll
    for (int e = 0; e < W; ++e) dot += acc[e] * acc[e];
    return dot;
}

// mean of one d = 3 query, sum over the 64 stencil nodes (one lane)
__device__ __forceinline__ double sorted3_mean(const Stencil& A, const double* __restrict__ amean, const GridDev& g,
                                               int base) {
    double mu = 0.0;
#pragma unroll 4
    for (int l = 0; l < 64; ++l) {
        const double w = A.w[0][l >> 4] * A.w[1][(l >> 2) & 3] * A.w[2][l & 3];
        mu += w * amean[base + (l >> 4) * g.stride[0] + ((l >> 2) & 3) * g.stride[1] + (l & 3)];
    }
    return mu;
}

// Queries counting-sorted by cell (SURVEY 8(f) NEXT #3a): a CTA stages the 64 stencil rows of
// cp.async of the 64 stencil rows of cell c (k_pad values each) into dst, one commit group
// TMA: the 64 rows are 16 runs of 4 consecutive nodes along the last axis, each run
// 4 k_pad contiguous values of the row-major Rc -- one cp.async.bulk per run, issued by one
// thread, completing on the buffer's mbarrier (expect_tx of the 64 rows' bytes)
template <typename V>
__device__ __forceinline__ void stage_rows3_tma(const GridDev& g, const V* __restrict__ Rc, int k_pad, int c, V* dst,
                                                uint64_t* bar) {
    if (threadIdx.x != 0) return;
    // the buffer was last read through the generic proxy (ordered by the __syncthreads that
    // ended that cell): order those reads before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    const int base = c - g.stride[0] - g.stride[1] - 1;
    const unsigned run = 4u * (unsigned)k_pad * (unsigned)sizeof(V);
    mbar_expect_tx(bar, 16u * run);
#pragma unroll
    for (int ab = 0; ab < 16; ++ab) {
        const int node = base + (ab >> 2) * g.stride[0] + (ab & 3) * g.stride[1];
        bulk_g2s(dst + (size_t)ab * 4 * k_pad, Rc + (int64_t)node * k_pad, run, bar);
    }
}

template <typename V>
__device__ __forceinline__ void stage_rows3(const GridDev& g, const V* __restrict__ Rc, int k_pad, int nch, int c,
                                            V* dst) {
    constexpr int W = QV<V>::W;
    const int base = c - g.stride[0] - g.stride[1] - 1;
    for (int e = threadIdx.x; e < 64 * nch; e += blockDim.x) {
        const int l = e / nch, ch = e - l * nch;
        const int node = base + (l >> 4) * g.stride[0] + ((l >> 2) & 3) * g.stride[1] + (l & 3);
        __pipeline_memcpy_async(dst + l * k_pad + ch * W, Rc + (int64_t)node * k_pad + ch * W, sizeof(V) * W);
    }
    __pipeline_commit();
}

// Rc of a cell in shared memory once.  Cells with at least kLanePerQuery queries: one lane per
// query, every lane reading the same row chunk (a shared-memory broadcast feeds 32 queries);
// sparser cells: a warp per query, lanes over 16-byte chunks of k.
constexpr int kLanePerQuery = 16;
constexpr bool kSorted3Tma = LOVE_SORTED3_TMA;   // row staging by cp.async.bulk (else per-thread cp.async)

#ifndef LOVE_SORTED3_MINB
#define LOVE_SORTED3_MINB 4   // measured: 1 CTA per SM at 168 registers 5.5 ms, 3 CTAs 3.24 ms, 4 CTAs (64 registers, small spills) 3.15 ms per 4e6 queries
#endif
// The stencil weights of a lane-mode query in the form the fp32 chunk loop uses, made once per
// query instead of once per chunk (the Stencil itself lives in local memory at 64 registers)
struct Q3W {
    f32x2 c[4];      // (w2[c], w2[c])
    f32x2 b[4];      // (w1[b], w1[b])
    double a[4];     // w0[a]
};
__device__ __forceinline__ Q3W make_q3w(const Stencil& A) {
    Q3W w;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float c = (float)A.w[2][i], b = (float)A.w[1][i];
        w.c[i] = pk2(c, c);
        w.b[i] = pk2(b, b);
        w.a[i] = A.w[0][i];
    }
    return w;
}
// the same FMAs in the same order as sorted3_chunk's fp32 path
__device__ __forceinline__ double sorted3_chunk_w(const Q3W& w, const float* rows, int k_pad, int ch) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        f32x2 ra01 = 0ull, ra23 = 0ull;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            f32x2 rb01 = 0ull, rb23 = 0ull;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const float4 v = *reinterpret_cast<const float4*>(rows + (a * 16 + b * 4 + cc) * k_pad + ch * 4);
                rb01 = fma2(w.c[cc], pk2(v.x, v.y), rb01);
                rb23 = fma2(w.c[cc], pk2(v.z, v.w), rb23);
            }
            ra01 = fma2(w.b[b], rb01, ra01);
            ra23 = fma2(w.b[b], rb23, ra23);
        }
        acc[0] += w.a[a] * (double)lo2(ra01);
        acc[1] += w.a[a] * (double)hi2(ra01);
        acc[2] += w.a[a] * (double)lo2(ra23);
        acc[3] += w.a[a] * (double)hi2(ra23);
    }
    double dot = 0.0;
#pragma unroll
    for (int e = 0; e < 4; ++e) dot += acc[e] * acc[e];
    return dot;
}
template <typename V>
__device__ __forceinline__ double sorted3_dot(const Stencil& A, const V* rows, int k_pad, int ch0, int nch, int step) {
    double dot = 0.0;
    if constexpr (sizeof(V) == 4 && LOVE_PAIRED_Q3 && kSorted3Hoist) {
        const Q3W w = make_q3w(A);
        for (int ch = ch0; ch < nch; ch += step) dot += sorted3_chunk_w(w, rows, k_pad, ch);
    } else {
        for (int ch = ch0; ch < nch; ch += step) dot += sorted3_chunk<V>(A, rows, k_pad, ch);
    }
    return dot;
}

template <typename V, int TPB = 256>
__global__ void __launch_bounds__(TPB, TPB == 256 ? LOVE_SORTED3_MINB : 4) predict_sorted3_kernel(GridDev g, C4 c4, double s2, double l0, double l1,
                                                              double l2, int prior_mode, const V* __restrict__ Rc,
                                                              int k_pad, const double* __restrict__ amean,
                                                              const double* __restrict__ Xs,
                                                              const int* __restrict__ qstart,
                                                              const int* __restrict__ perm, int cells_per_cta,
                                                              V* __restrict__ out, V* __restrict__ mean_out,
                                                              unsigned long long* __restrict__ counters,
                                                              int lane_mode_min) {
    constexpr int W = QV<V>::W;
    using VT = typename QV<V>::T;
    extern __shared__ __align__(16) unsigned char smraw[];
    // two [64][k_pad] row buffers: the rows of the next occupied cell are copied in
    // (cp.async, no registers) while the queries of the current one are answered
    V* const rows0 = reinterpret_cast<V*>(smraw);
    const int64_t bstride = 64 * (int64_t)k_pad;
    __shared__ double part[256];                                 // lane mode: [warp][lane] partial norms
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nch = k_pad / W;
    const int m = g.m_total;
    const int c_begin = blockIdx.x * cells_per_cta;
    const int c_end = min(m, c_begin + cells_per_cta);
    __shared__ __align__(8) uint64_t bars[2];                   // TMA completion, one per buffer
    unsigned phase[2] = {0u, 0u};
    if (kSorted3Tma && threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init_fence();
    }
    if (kSorted3Tma) __syncthreads();
    int c = c_begin;
    while (c < c_end && qstart[c] == qstart[c + 1]) ++c;        // first cell with queries
    if (c < c_end) {
        if (kSorted3Tma) stage_rows3_tma<V>(g, Rc, k_pad, c, rows0, &bars[0]);
        else stage_rows3<V>(g, Rc, k_pad, nch, c, rows0);
    }
    int buf = 0;
    while (c < c_end) {
        int cn = c + 1;
        while (cn < c_end && qstart[cn] == qstart[cn + 1]) ++cn;
        if (kSorted3Tma) {
            if (cn < c_end) stage_rows3_tma<V>(g, Rc, k_pad, cn, rows0 + (buf ^ 1) * bstride, &bars[buf ^ 1]);
            mbar_wait(&bars[buf], phase[buf]);                  // this cell's rows have landed
            phase[buf] ^= 1u;
        } else {
            if (cn < c_end) stage_rows3<V>(g, Rc, k_pad, nch, cn, rows0 + (buf ^ 1) * bstride);
            if (cn < c_end) __pipeline_wait_prior(1);            // this cell's rows have landed
            else __pipeline_wait_prior(0);
        }
        __syncthreads();
        const V* rows = rows0 + buf * bstride;
        const int p0 = qstart[c], p1 = qstart[c + 1];
        const int base = c - g.stride[0] - g.stride[1] - 1;      // node of stencil offset (0, 0, 0)
        const int nq = p1 - p0;
        if (nq >= lane_mode_min) {                              // lane per query
            // groups of 32 queries; with fewer groups than warps, wpg warps share a group and
            // split its k chunks (partial norms combined in shared memory)
            const int groups = (nq + 31) >> 5;
            // whole rounds of nw groups: a warp per group of 32; the remaining groups (fewer than
            // nw) share the warps below, splitting k (no round with idle warps at the barrier)
            const int full = kSorted3Balance ? groups / nw * nw : (groups >= nw ? groups : 0);
            for (int gi = wid; gi < full; gi += nw) {
                const int pos = p0 + gi * 32 + lane;
                if (pos >= p1) continue;
                const int q = perm[pos];
                const Stencil A = make_stencil<3>(g, Xs + (int64_t)q * 3);
                const double dot = sorted3_dot<V>(A, rows, k_pad, 0, nch, 1);
                finish_sorted3<V>(A, c4, s2, prior_mode, dot,
                                  mean_out ? sorted3_mean(A, amean, g, base) : 0.0, q, out, mean_out, counters);
            }
            if (groups > full) {                                // wpg warps per group: split k
                const int rem = groups - full;
                const int wpg = nw / rem;
                const int gi = full + wid / wpg, sub = wid - (wid / wpg) * wpg;
                const int pos = p0 + gi * 32 + lane;
                const bool live = gi < groups && pos < p1;
                const int q = live ? perm[pos] : 0;
                Stencil A;
                double dot = 0.0;
                if (live) {
                    A = make_stencil<3>(g, Xs + (int64_t)q * 3);
                    dot = sorted3_dot<V>(A, rows, k_pad, sub, nch, wpg);
                }
                part[wid * 32 + lane] = dot;                    // [warp][lane]
                __syncthreads();
                if (live && sub == 0) {
                    for (int t = 1; t < wpg; ++t) dot += part[(wid + t) * 32 + lane];
                    finish_sorted3<V>(A, c4, s2, prior_mode, dot,
                                      mean_out ? sorted3_mean(A, amean, g, base) : 0.0, q, out, mean_out, counters);
                }
            }
            __syncthreads();
            c = cn;
            buf ^= 1;
            continue;
        }
        for (int pos = p0 + wid; pos < p1; pos += nw) {         // warp per query
            const int q = perm[pos];
            const Stencil A = make_stencil<3>(g, Xs + (int64_t)q * 3);
            double dot = 0.0;
            for (int ch = lane; ch < nch; ch += 32) dot += sorted3_chunk<V>(A, rows, k_pad, ch);
            // mean: each lane takes 2 of the 64 nodes
            double mu = 0.0;
            if (mean_out) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int l = lane + 32 * h;
                    const double w = pick4(A.w[0], l >> 4) * pick4(A.w[1], (l >> 2) & 3) * pick4(A.w[2], l & 3);
                    mu += w * amean[base + (l >> 4) * g.stride[0] + ((l >> 2) & 3) * g.stride[1] + (l & 3)];
                }
                mu = warp_sum(mu);
            }
            dot = warp_sum(dot);
            if (lane != 0) continue;
            finish_sorted3<V>(A, c4, s2, prior_mode, dot, mu, q, out, mean_out, counters);
        }
        __syncthreads();                                        // this buffer is free for cell cn + 1
        c = cn;
        buf ^= 1;
    }
}

template <typename V>
__global__ void nan_fill_kernel(const int* __restrict__ qstart, int m, const int* __restrict__ perm,
                                V* __restrict__ out, V* __restrict__ mean_out,
                                unsigned long long* __restrict__ counters) {
    const int p0 = qstart[m], p1 = qstart[m + 1];
    for (int pos = p0 + blockIdx.x * blockDim.x + threadIdx.x; pos < p1; pos += gridDim.x * blockDim.x) {
        const int q = perm[pos];
        out[q] = (V)NAN;
        if (mean_out) mean_out[q] = (V)NAN;
        atomicAdd(&counters[1], 1ull);
    }
}

// opt-in shared memory per block of the current device, and the static shared memory of the
// sorted d = 3 kernel (both host queries, cached)
size_t optin_smem() {
    int dev = 0, v = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem optin");
    return (size_t)v;
}

template <typename V>
size_t sorted3_static_smem() {
    static size_t bytes = 0;
    if (bytes == 0) {
        cudaFuncAttributes a{};
        cuda_check(cudaFuncGetAttributes(&a, (const void*)predict_sorted3_kernel<V>), "func attributes");
        bytes = a.sharedSizeBytes + 1;
    }
    return bytes - 1;
}

void build_var_blocks(Cache& c, cudaStream_t s) {
    if (c.additive || c.g.d > 2 || c.var_blocks_off || c.k_eff < 1) return;
    ProfScope ps(LOVE_PROF_FINISH, s);
    const int m = c.g.m_total;
    c.vblk = dalloc(c, sizeof(double) * (size_t)m * blk_size(c.g.d), s);
    if (c.g.d == 1)
        LOVE_LAUNCH(var_blocks1_kernel, (int)ceil_div(m, 256), 256, 0, s, m, c.k_eff, (const double*)c.Rc_col,
                    (const double*)c.cols64, c.rbf.outputscale, (double*)c.vblk);
    else if (std::getenv("LOVE_VAR_BLOCKS2_WARP") != nullptr)   // the warp-per-cell kernel (cross-check)
        LOVE_LAUNCH(var_blocks2_kernel, (int)ceil_div((int64_t)m * 32, 256), 256, 0, s, c.g, c.k_eff,
                    (const double*)c.Rc_col, (const double*)c.cols64, c.rbf.outputscale, (double*)c.vblk);
    else {
        double* P = nullptr;
        cuda_check(cudaMallocAsync((void**)&P, sizeof(double) * kPairOffs * (size_t)m, s), "pair products");
        const dim3 grid((unsigned)ceil_div(c.g.m[1], kPTJ), (unsigned)ceil_div(c.g.m[0], kPTI));
        LOVE_LAUNCH(pair_products2_kernel, grid, kPTI * kPTJ, 0, s, c.g, c.k_eff, (const double*)c.Rc_col, P);
        LOVE_LAUNCH(assemble_blocks2_kernel, (int)ceil_div((int64_t)m * 136, 256), 256, 0, s, c.g, (const double*)P,
                    (const double*)c.cols64, c.rbf.outputscale, (double*)c.vblk);
        cuda_check(cudaFreeAsync(P, s), "pair products free");
    }
}

template <typename V>
void launch_predict(const Cache& c, const double* Xa, const double* Xb, int64_t t, V* out, V* mean_out,
                    cudaStream_t s) {
    if (t <= 0) return;
    ProfScope ps(LOVE_PROF_QUERY, s);
    if (c.additive) {
        add_predict<V>(c, Xa, Xb, t, out, mean_out, s);
        return;
    }
    if (Xb == nullptr && c.vblk != nullptr) {
        C4 c4{};
        for (int d = 0; d < c.g.d; ++d)
            for (int e = 0; e < 4; ++e) c4.c[d][e] = c.h_cols64[d][e];
        const char* ce = std::getenv("LOVE_QUERY_COOP");
        const bool coop = ce == nullptr || std::atoi(ce) != 0;
        // measured (ncu, 10^6 queries): d = 2 with 8 lanes per query 245 vs 348 us; d = 1 keeps
        // one thread per query (25 vs 32 us with 2 lanes)
        if (coop && c.g.d == 2) {                // G lanes per query (d = 2: 8)
            if (c.g.d == 1)
                LOVE_LAUNCH((predict_block_coop_kernel<V, 1, 2>), (int)ceil_div(t, 128), 256, 0, s, c.g, c4,
                            c.rbf.outputscale, c.prior, (const double*)c.vblk, (const double*)c.a, Xa, t, out, mean_out,
                            c.counters);
            else
                LOVE_LAUNCH((predict_block_coop_kernel<V, 2, 8>), (int)ceil_div(t, 32), 256, 0, s, c.g, c4,
                            c.rbf.outputscale, c.prior, (const double*)c.vblk, (const double*)c.a, Xa, t, out, mean_out,
                            c.counters);
            return;
        }
        // one query per thread (measured: two per thread with interleaved chains is ~8% slower)
        if (c.g.d == 1)
            LOVE_LAUNCH((predict_block_kernel<V, 1, 1>), (int)ceil_div(t, 256), 256, 0, s, c.g, c4, c.rbf.outputscale,
                        c.prior, (const double*)c.vblk, (const double*)c.a, Xa, t, out, mean_out, c.counters);
        else
            LOVE_LAUNCH((predict_block_kernel<V, 2, 1>), (int)ceil_div(t, 256), 256, 0, s, c.g, c4, c.rbf.outputscale,
                        c.prior, (const double*)c.vblk, (const double*)c.a, Xa, t, out, mean_out, c.counters);
        return;
    }
    // d = 3 cell-sorted path: the 64 stencil rows of a cell (64 k_pad values) must fit in one
    // CTA's shared memory next to the kernel's static arrays; larger k takes the per-query path
    const size_t sm3 = 2 * sizeof(V) * 64 * (size_t)c.k_pad;   // two row buffers
    if (Xb == nullptr && c.g.d == 3 && t >= 65536 && std::getenv("LOVE_NO_SORTED_QUERIES") == nullptr &&
        sm3 + sorted3_static_smem<V>() <= optin_smem()) {
        const int m = c.g.m_total;
        struct Tmp {                                    // freed on every exit (stream-ordered)
            cudaStream_t s;
            int *key = nullptr, *perm = nullptr, *qstart = nullptr;
            ~Tmp() {
                if (key) cudaFreeAsync(key, s);
                if (perm) cudaFreeAsync(perm, s);
                if (qstart) cudaFreeAsync(qstart, s);
            }
        } tm{s};
        cuda_check(cudaMallocAsync((void**)&tm.key, sizeof(int) * t, s), "query sort alloc");
        cuda_check(cudaMallocAsync((void**)&tm.perm, sizeof(int) * t, s), "query sort alloc");
        cuda_check(cudaMallocAsync((void**)&tm.qstart, sizeof(int) * (m + 2), s), "query sort alloc");
        LOVE_LAUNCH(query_cell3_kernel, (int)std::min<int64_t>(ceil_div(t, 256), 148 * 16), 256, 0, s, c.g, Xa, t,
                    tm.key);
        counting_sort_keys(tm.key, t, m + 1, tm.qstart, tm.perm, s);
        C4 c4{};
        for (int d = 0; d < 3; ++d)
            for (int e = 0; e < 4; ++e) c4.c[d][e] = c.h_cols64[d][e];
        // cells per CTA and the lane-mode threshold (measurement switches LOVE_Q3_CPC / LOVE_Q3_LMIN)
        static const int cpc = std::getenv("LOVE_Q3_CPC") ? std::max(1, std::atoi(std::getenv("LOVE_Q3_CPC"))) : 8;
        static const int lmin = std::getenv("LOVE_Q3_LMIN") ? std::max(1, std::atoi(std::getenv("LOVE_Q3_LMIN")))
                                                            : kLanePerQuery;
        // 4 warps per CTA (LOVE_Q3_TPB=256: 8): the per-cell barrier idles fewer warps in the many
        // cells with few queries, and 128 registers drop the 64-register spills; measured cfg4
        // 27.50 -> 27.19 ms (same box, three interleaved repeats)
        static const int tpb = std::getenv("LOVE_Q3_TPB") ? std::atoi(std::getenv("LOVE_Q3_TPB")) : 128;
        if (tpb == 128) {
            ensure_smem((const void*)predict_sorted3_kernel<V, 128>, sm3);
            LOVE_LAUNCH((predict_sorted3_kernel<V, 128>), (int)ceil_div(m, cpc), 128, sm3, s, c.g, c4, c.rbf.outputscale,
                        c.rbf.lengthscale[0], c.rbf.lengthscale[1], c.rbf.lengthscale[2], c.prior, (const V*)c.Rc,
                        c.k_pad, (const double*)c.a, Xa, tm.qstart, tm.perm, cpc, out, mean_out, c.counters, lmin);
        } else {
            ensure_smem((const void*)predict_sorted3_kernel<V>, sm3);
            LOVE_LAUNCH(predict_sorted3_kernel<V>, (int)ceil_div(m, cpc), 256, sm3, s, c.g, c4, c.rbf.outputscale,
                        c.rbf.lengthscale[0], c.rbf.lengthscale[1], c.rbf.lengthscale[2], c.prior, (const V*)c.Rc,
                        c.k_pad, (const double*)c.a, Xa, tm.qstart, tm.perm, cpc, out, mean_out, c.counters, lmin);
        }
        LOVE_LAUNCH(nan_fill_kernel<V>, 64, 256, 0, s, tm.qstart, m, tm.perm, out, mean_out, c.counters);
        return;
    }
    constexpr int G = 8;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(t, 8 * (32 / G)), 148 * 16));
    const double* L = c.rbf.lengthscale;
    C4 c4{};
    for (int d = 0; d < c.g.d; ++d)
        for (int e = 0; e < 4; ++e) c4.c[d][e] = c.h_cols64[d][e];
#define LOVE_PREDICT(DD)                                                                                         \
    LOVE_LAUNCH((predict_kernel<V, DD, G>), blocks, 256, 0, s, c.g, c.cols64, c4, c.rbf.outputscale, L[0], L[1],  \
                L[2], c.prior, (const V*)c.Rc, c.k_pad, (const double*)c.a, Xa, Xb, t, out, mean_out, c.counters)
    switch (c.g.d) {
        case 1: LOVE_PREDICT(1); break;
        case 2: LOVE_PREDICT(2); break;
        default: LOVE_PREDICT(3); break;
    }
#undef LOVE_PREDICT
}

template void launch_predict<float>(const Cache&, const double*, const double*, int64_t, float*, float*,
                                    cudaStream_t);
template void launch_predict<double>(const Cache&, const double*, const double*, int64_t, double*, double*,
                                     cudaStream_t);

}  // namespace love
