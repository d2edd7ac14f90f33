// ski.cu -- the sparse interpolation operators of the SKI MVM.
//
//   scatter  u = W_X q   (n -> m)   -- per-item stencil moments, then an atomic-free node pull
//   gather   r = W_X^T z + sigma^2 q, alpha = q^T r   (m -> n, fp64 alpha)
//
// Points are sorted by cell and cut into items of <= kItemMax points of one cell, so:
//  * scatter: one thread per item sums q_p * w_l(p) over its points into 4^d registers
//    ("moments" M[l][item]); one thread per grid node i then pulls M[l][item] from the items
//    of the 4^d cells whose stencil slot l lands on i.  No atomics (shared-memory float
//    atomics are CAS loops on sm_100a) and a deterministic summation order.
//  * gather: one thread per item loads the 4^d z values of its cell's stencil once and
//    reuses them for every point of the item.
#include <cuda_runtime.h>
#include <cstdlib>
#include <type_traits>

#include "love_internal.h"
#include "ski_device.cuh"

namespace love {

LOVE_TRACE_TU(ski)

namespace {

#ifndef LOVE_BATCH
#define LOVE_BATCH 8
#endif
constexpr int kBatch = LOVE_BATCH;   // points loaded per batch (memory-level parallelism)
#ifndef LOVE_PULL2_SG
#define LOVE_PULL2_SG 4     // outer slots per thread of the 2-D last-axis pull (4: one thread per node)
#endif
#ifndef LOVE_PULL3_SG
#define LOVE_PULL3_SG 4     // outer slots per thread of the 3-D last-axis pull (16: one thread per node)
#endif
#ifndef LOVE_PAIRED3
#define LOVE_PAIRED3 1
#endif
constexpr bool kPaired3 = LOVE_PAIRED3;   // 3-D fp32 moments on FFMA2 pairs
// the paired 3-D gather (two points per FFMA2) is bitwise identical but measured slower
// (cfg4 gather 3.98 -> 4.19 ms per build): off
constexpr bool kPairedGather3 = false;
// the 3-D fp32 gather with the stencil's b-pairs packed (z[a][b][c], z[a][b+1][c]): the 64 c-level
// FMAs of a point as 32 FFMA2, the same FMA per slot in the same order as stencil_dot<float, 3>
#ifndef LOVE_BPAIR_GATHER3
#define LOVE_BPAIR_GATHER3 1
#endif
constexpr bool kBPairGather3 = LOVE_BPAIR_GATHER3;

// minimum resident CTAs per SM for the 3-D item kernels (0: the compiler's choice)
#ifndef LOVE_MOM3_MINB
#define LOVE_MOM3_MINB 0
#endif
#ifndef LOVE_GATHER3_MINB
#define LOVE_GATHER3_MINB 0
#endif
#if LOVE_MOM3_MINB > 0
#define LOVE_MOM_BOUNDS(D) __launch_bounds__(256, (D) == 3 ? LOVE_MOM3_MINB : 1)
#else
#define LOVE_MOM_BOUNDS(D) __launch_bounds__(256)
#endif
#if LOVE_GATHER3_MINB > 0
#define LOVE_GATHER_BOUNDS(D) __launch_bounds__(256, (D) == 3 ? LOVE_GATHER3_MINB : 1)
#else
#define LOVE_GATHER_BOUNDS(D) __launch_bounds__(256)
#endif
// LOVE_TAIL_BREAK: the compute loop of a point batch stops at the item's end instead of running
// the zero-weighted padding of the last batch (cfg4 in-graph: moments 29.8 -> 25.4 us per step)
#ifndef LOVE_TAIL_BREAK
#define LOVE_TAIL_BREAK 1
#endif
#if LOVE_TAIL_BREAK
#define LOVE_BATCH_END(cond) if (cond) break
#else
#define LOVE_BATCH_END(cond) (void)0
#endif

template <typename V, int D, typename MT>
__global__ void LOVE_MOM_BOUNDS(D) moments_kernel(int64_t n_items, const int* __restrict__ item_start,
                                                      const V* __restrict__ f0, const V* __restrict__ f1,
                                                      const V* __restrict__ f2, const V* __restrict__ qbase,
                                                      StepRef ref, MT* __restrict__ M) {
    pdl_wait();
    LOVE_TRACE(kTrMoments, step_j(ref));
    using A = typename AccT<V, D>::type;
    constexpr int S = Slots<D>::value;
    const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (it >= n_items || step_done(ref)) return;
    const V* __restrict__ q = qbase + step_j(ref) * ref.ld;
    const int p0 = item_start[it], p1 = item_start[it + 1];
    if constexpr (D == 3 && std::is_same<A, float>::value && kPaired3) {
        // accumulators in pairs (slots c, c + 1 of one (a, b)): one FFMA2 per pair, the
        // point's (a, b) factor broadcast; the same FMA per slot as stencil_accum
        f32x2 acc2[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) acc2[l] = 0ull;
        for (int pb = p0; pb < p1; pb += kBatch) {
            float qv[kBatch], fa[kBatch], fb[kBatch], fc[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int p = pb + u;
                const bool in = p < p1;
                qv[u] = in ? (float)q[p] : 0.f;
                fa[u] = in ? (float)f0[p] : 0.f;
                fb[u] = in ? (float)f1[p] : 0.f;
                fc[u] = in ? (float)f2[p] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                LOVE_BATCH_END(pb + u >= p1);
                float w0[4], w1[4], w2[4];
                keys4<float>(fa[u], w0);
                keys4<float>(fb[u], w1);
                keys4<float>(fc[u], w2);
                const f32x2 w2lo = pk2(w2[0], w2[1]), w2hi = pk2(w2[2], w2[3]);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const float ta = qv[u] * w0[a];
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const float tb = ta * w1[b];
                        const f32x2 tt = pk2(tb, tb);
                        acc2[(a * 4 + b) * 2] = fma2(tt, w2lo, acc2[(a * 4 + b) * 2]);
                        acc2[(a * 4 + b) * 2 + 1] = fma2(tt, w2hi, acc2[(a * 4 + b) * 2 + 1]);
                    }
                }
            }
        }
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            M[(int64_t)(2 * l) * n_items + it] = (MT)lo2(acc2[l]);
            M[(int64_t)(2 * l + 1) * n_items + it] = (MT)hi2(acc2[l]);
        }
        return;
    }
    A acc[S];
#pragma unroll
    for (int l = 0; l < S; ++l) acc[l] = A(0);
    for (int pb = p0; pb < p1; pb += kBatch) {
        A qv[kBatch], fa[kBatch], fb[kBatch], fc[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int p = pb + u;
            const bool in = p < p1;
            qv[u] = in ? (A)q[p] : A(0);    // q = 0 makes padded lanes contribute nothing
            fa[u] = in ? (A)f0[p] : A(0);
            fb[u] = (D > 1 && in) ? (A)f1[p] : A(0);
            fc[u] = (D > 2 && in) ? (A)f2[p] : A(0);
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            A w0[4], w1[4], w2[4];
            keys4<A>(fa[u], w0);
            if (D > 1) keys4<A>(fb[u], w1);
            if (D > 2) keys4<A>(fc[u], w2);
            stencil_accum<A, D>(acc, qv[u], w0, w1, w2);
        }
    }
#pragma unroll
    for (int l = 0; l < S; ++l) M[(int64_t)l * n_items + it] = (MT)acc[l];
}

// d = 2 item moments with two lanes per item (interleaved points, one load batch each,
// combined by a shuffle): the 16 fp64 accumulators of an item of ~8 points in half the chain
template <typename V>
__global__ void __launch_bounds__(256) moments2_tpc_kernel(int64_t n_items, const int* __restrict__ item_start,
                                                           const V* __restrict__ f0, const V* __restrict__ f1,
                                                           const V* __restrict__ qbase, StepRef ref,
                                                           double* __restrict__ M) {
    pdl_wait();
    LOVE_TRACE(kTrMoments, step_j(ref));
    constexpr int B = 4;
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t it = gt >> 1;
    const int sub = (int)(gt & 1);
    if (step_done(ref)) return;
    const bool live = it < n_items;
    const V* __restrict__ q = qbase + step_j(ref) * ref.ld;
    const int p0 = live ? item_start[it] : 0, p1 = live ? item_start[it + 1] : 0;
    double acc[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) acc[l] = 0.0;
    for (int pb = p0 + sub; pb < p1; pb += 2 * B) {
        double qv[B], fa[B], fb[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int p = pb + 2 * u;
            const bool in = p < p1;
            qv[u] = in ? (double)q[p] : 0.0;
            fa[u] = in ? (double)f0[p] : 0.0;
            fb[u] = in ? (double)f1[p] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            LOVE_BATCH_END(pb + 2 * u >= p1);
            double w0[4], w1[4];
            keys4<double>(fa[u], w0);
            keys4<double>(fb[u], w1);
            stencil_accum<double, 2>(acc, qv[u], w0, w1, w1);
        }
    }
#pragma unroll
    for (int l = 0; l < 16; ++l) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], 1);
    if (!live || sub != 0) return;
#pragma unroll
    for (int l = 0; l < 16; ++l) M[(int64_t)l * n_items + it] = acc[l];
}

// ---- separable node pull of the scatter (d >= 2), u = W q from the per-item moments
// M[l][item], slot l = ((a*4 + b)*4 + c) (d = 3) or a*4 + b (d = 2), last index along the
// last grid axis.  Node (i_0, .., i_{d-1}) receives slot component s_e from cell i_e - s_e + 1
// along axis e, so the pull factorises axis by axis:
//   pull_last : T[so][lead cells, i_last] = sum_c sum_{items of cell (lead, i_last - c + 1)} M[so*4 + c][item]
//   pull_mid  : V[a][c0, i1, i2]          = sum_b T[a*4 + b][c0, i1 - b + 1, i2]          (d = 3)
//   pull_first: u[i0, ...]                = s_j * sum_a X[a][i0 - a + 1, ...]            (X = V or T)
// Every pull reads 4 neighbours per output, coalesced along the last axis.
// Thread per (node x, group of SG outer slots): d = 3 has 16 outer slots so, split over
// 16 / SG threads per node (x fastest: coalesced M and T along the grid), fewer registers
// and shorter chains per thread than one thread per node.
template <int D, typename MT, int SG, typename TT = double>
__global__ void __launch_bounds__(256) pull_last_kernel(GridDev g, int64_t n_items, const int* __restrict__ cis,
                                                        const MT* __restrict__ M, StepRef ref,
                                                        TT* __restrict__ T) {
    pdl_wait();
    LOVE_TRACE(kTrPullLast, step_j(ref));
    constexpr int SO = D == 2 ? 4 : 16;
    static_assert(SO % SG == 0, "slot groups");
    const int m = g.m_total;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= (int64_t)m * (SO / SG) || step_done(ref)) return;
    const int grp = (int)(idx / m), x = (int)(idx - (int64_t)grp * m);
    const int so0 = grp * SG;
    const int ml = g.m[D - 1];
    const int il = x % ml;
    double sum[SG];
#pragma unroll
    for (int so = 0; so < SG; ++so) sum[so] = 0.0;
    if constexpr (D == 3) {   // (the batched form below measured slower here: cfg4 +0.4 ms)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int cl = il - c + 1;
            if (cl < 0 || cl >= ml) continue;
            const int cell = x + 1 - c;
            const int e = cis[cell + 1];
            for (int it = cis[cell]; it < e; ++it)
#pragma unroll
                for (int so = 0; so < SG; ++so) sum[so] += (double)M[(int64_t)((so0 + so) * 4 + c) * n_items + it];
        }
#pragma unroll
        for (int so = 0; so < SG; ++so) T[(int64_t)(so0 + so) * m + x] = (TT)sum[so];
        return;
    }
    // d = 2: the four cells' item ranges first, then the first item of every cell (4 SG
    // independent loads in flight), then the rare further items; summed in the original order
    // (c, item): cfg3 8.04 -> 7.96 ms
    int ib[4], ie[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int cl = il - c + 1;
        const bool ok = cl >= 0 && cl < ml;
        ib[c] = ok ? cis[x + 1 - c] : 0;
        ie[c] = ok ? cis[x + 2 - c] : 0;
    }
    MT v[4][SG];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int so = 0; so < SG; ++so)
            v[c][so] = ie[c] > ib[c] ? M[(int64_t)((so0 + so) * 4 + c) * n_items + ib[c]] : MT(0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        if (ie[c] <= ib[c]) continue;
#pragma unroll
        for (int so = 0; so < SG; ++so) sum[so] += (double)v[c][so];
        for (int it = ib[c] + 1; it < ie[c]; ++it)
#pragma unroll
            for (int so = 0; so < SG; ++so) sum[so] += (double)M[(int64_t)((so0 + so) * 4 + c) * n_items + it];
    }
#pragma unroll
    for (int so = 0; so < SG; ++so) T[(int64_t)(so0 + so) * m + x] = sum[so];
}

__global__ void __launch_bounds__(256) pull_mid_kernel(GridDev g, const double* __restrict__ T, StepRef ref,
                                                       double* __restrict__ Vout) {
    pdl_wait();
    LOVE_TRACE(kTrPullMid, step_j(ref));
    const int m = g.m_total;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= 4 * (int64_t)m || step_done(ref)) return;
    const int a = (int)(idx / m), x = (int)(idx - (int64_t)a * m);
    const int i1 = (x / g.stride[1]) % g.m[1];
    double sum = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int c1 = i1 - b + 1;
        if (c1 < 0 || c1 >= g.m[1]) continue;
        sum += T[(int64_t)(a * 4 + b) * m + x + (1 - b) * g.stride[1]];
    }
    Vout[idx] = sum;
}

__global__ void __launch_bounds__(256) pull_first_kernel(GridDev g, const double* __restrict__ X, StepRef ref,
                                                         double* __restrict__ u) {
    pdl_wait();
    LOVE_TRACE(kTrPullFirst, step_j(ref));
    const int m = g.m_total;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= m || step_done(ref)) return;
    const int i0 = x / g.stride[0];
    double sum = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int c0 = i0 - a + 1;
        if (c0 < 0 || c0 >= g.m[0]) continue;
        sum += X[(int64_t)a * m + x + (1 - a) * g.stride[0]];
    }
    u[x] = sum * ref.scale[step_j(ref)];
}

// d = 3: pull_mid and pull_first in one pass (each T entry is read by exactly one node):
//   u[i0, i1, i2] = s_j * sum_a ( sum_b T[a*4 + b][i0 - a + 1, i1 - b + 1, i2] )
// with the same two summation orders as the separate passes (bitwise the same u)
template <typename TT>
__global__ void __launch_bounds__(256) pull_mid_first_kernel(GridDev g, const TT* __restrict__ T, StepRef ref,
                                                             double* __restrict__ u) {
    pdl_wait();
    LOVE_TRACE(kTrPullMid, step_j(ref));
    const int m = g.m_total;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= m || step_done(ref)) return;
    const int i0 = x / g.stride[0];
    const int i1 = (x / g.stride[1]) % g.m[1];
    double sum = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int c0 = i0 - a + 1;
        if (c0 < 0 || c0 >= g.m[0]) continue;
        const int64_t xa = x + (int64_t)(1 - a) * g.stride[0];
        double va = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int c1 = i1 - b + 1;
            if (c1 < 0 || c1 >= g.m[1]) continue;
            va += (double)T[(int64_t)(a * 4 + b) * m + xa + (1 - b) * g.stride[1]];
        }
        sum += va;
    }
    u[x] = sum * ref.scale[step_j(ref)];
}

// u[i] = scale * sum over slots l of sum over items of cell (i - l + 1) of M[l][item]
template <int D>
__global__ void __launch_bounds__(256) nodepass_kernel(GridDev g, int64_t n_items,
                                                       const int* __restrict__ cis,
                                                       const double* __restrict__ M, StepRef ref,
                                                       double* __restrict__ u) {
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.m_total || step_done(ref)) return;
    u[i] = node_pull<D>(g, n_items, cis, M, i) * ref.scale[step_j(ref)];
}

template <typename V, int D>
__global__ void LOVE_GATHER_BOUNDS(D) gather_kernel(GridDev g, int64_t n_items,
                                                     const int* __restrict__ item_cell,
                                                     const int* __restrict__ item_start,
                                                     const V* __restrict__ f0, const V* __restrict__ f1,
                                                     const V* __restrict__ f2, const double* __restrict__ z,
                                                     const V* __restrict__ qbase, StepRef ref, double sigma2,
                                                     V* __restrict__ r, double* __restrict__ alpha_base,
                                                     RcStream rs, int ngather) {
    pdl_wait();
    LOVE_TRACE(kTrGather, step_j(ref));
    if ((int)blockIdx.x >= ngather) {          // extra CTAs: the streamed cache column (last: the
        // d >= 2 gather is the longer job, its CTAs go first)
        stream_rc_column(rs, (blockIdx.x - ngather) * blockDim.x + threadIdx.x, (gridDim.x - ngather) * blockDim.x);
        return;
    }
    using A = typename AccT<V, D>::type;
    constexpr int S = Slots<D>::value;
    __shared__ double red[32];
    const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (step_done(ref)) return;
    const int j = step_j(ref);
    const V* __restrict__ q = qbase + j * ref.ld;
    const double sc = ref.scale[j];
    const A vsc = (A)sc, vsig = (A)(sigma2 * sc);
    double alpha = 0.0;
    if constexpr (D == 3 && std::is_same<A, float>::value && kBPairGather3) {
        if (it < n_items) {
            f32x2 zp[32];                          // [a][b pair][c]
            {
                float zl[64];
                load_stencil<float, 3>(g, z, stencil_base<3>(g, item_cell[it]), zl);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int bp = 0; bp < 2; ++bp)
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc)
                            zp[(a * 2 + bp) * 4 + cc] = pk2(zl[(a * 4 + 2 * bp) * 4 + cc], zl[(a * 4 + 2 * bp + 1) * 4 + cc]);
            }
            const int p0 = item_start[it], p1 = item_start[it + 1];
            for (int pb = p0; pb < p1; pb += kBatch) {
                float qv[kBatch], fa[kBatch], fb[kBatch], fc[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int p = pb + u;
                    const bool in = p < p1;
                    qv[u] = in ? (float)q[p] : 0.f;
                    fa[u] = in ? (float)f0[p] : 0.f;
                    fb[u] = in ? (float)f1[p] : 0.f;
                    fc[u] = in ? (float)f2[p] : 0.f;
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    LOVE_BATCH_END(pb + u >= p1);
                    float w0[4], w1[4], w2[4];
                    keys4<float>(fa[u], w0);
                    keys4<float>(fb[u], w1);
                    keys4<float>(fc[u], w2);
                    float acc = 0.f;
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        f32x2 t01 = 0ull, t23 = 0ull;      // (tb[a][0], tb[a][1]), (tb[a][2], tb[a][3])
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) {
                            const f32x2 ww = pk2(w2[cc], w2[cc]);
                            t01 = fma2(ww, zp[(a * 2) * 4 + cc], t01);
                            t23 = fma2(ww, zp[(a * 2 + 1) * 4 + cc], t23);
                        }
                        float ta = 0.f;
                        ta = fmaf(w1[0], lo2(t01), ta);
                        ta = fmaf(w1[1], hi2(t01), ta);
                        ta = fmaf(w1[2], lo2(t23), ta);
                        ta = fmaf(w1[3], hi2(t23), ta);
                        acc = fmaf(w0[a], ta, acc);
                    }
                    const V rv = (V)(acc + vsig * qv[u]);
                    if (pb + u < p1) {
                        r[pb + u] = rv;
                        alpha += (double)(vsc * qv[u]) * (double)rv;
                    }
                }
            }
        }
    } else if (it < n_items) {
        A zl[S];
        load_stencil<A, D>(g, z, stencil_base<D>(g, item_cell[it]), zl);
        const int p0 = item_start[it], p1 = item_start[it + 1];
        for (int pb = p0; pb < p1; pb += kBatch) {
            A qv[kBatch], fa[kBatch], fb[kBatch], fc[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int p = pb + u;
                const bool in = p < p1;
                qv[u] = in ? (A)q[p] : A(0);
                fa[u] = in ? (A)f0[p] : A(0);
                fb[u] = (D > 1 && in) ? (A)f1[p] : A(0);
                fc[u] = (D > 2 && in) ? (A)f2[p] : A(0);
            }
            if constexpr (D == 3 && std::is_same<A, float>::value && kPairedGather3) {
#pragma unroll
                for (int u = 0; u < kBatch; u += 2) {          // two points per FFMA2
                    float wa[4], wb[4], ua[4], ub[4], va[4], vb[4];
                    keys4<float>(fa[u], wa);
                    keys4<float>(fa[u + 1], wb);
                    keys4<float>(fb[u], ua);
                    keys4<float>(fb[u + 1], ub);
                    keys4<float>(fc[u], va);
                    keys4<float>(fc[u + 1], vb);
                    f32x2 w0[4], w1[4], w2[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        w0[i] = pk2(wa[i], wb[i]);
                        w1[i] = pk2(ua[i], ub[i]);
                        w2[i] = pk2(va[i], vb[i]);
                    }
                    const f32x2 d2 = stencil_dot3_pair(w0, w1, w2, zl);
                    const float rv0 = lo2(d2) + vsig * qv[u], rv1 = hi2(d2) + vsig * qv[u + 1];
                    if (pb + u < p1) {
                        r[pb + u] = (V)rv0;
                        alpha += (double)(vsc * qv[u]) * (double)(V)rv0;
                    }
                    if (pb + u + 1 < p1) {
                        r[pb + u + 1] = (V)rv1;
                        alpha += (double)(vsc * qv[u + 1]) * (double)(V)rv1;
                    }
                }
            } else {
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                if (D == 3) LOVE_BATCH_END(pb + u >= p1);
                A w0[4], w1[4], w2[4];
                keys4<A>(fa[u], w0);
                if (D > 1) keys4<A>(fb[u], w1);
                if (D > 2) keys4<A>(fc[u], w2);
                const V rv = (V)(stencil_dot<A, D>(w0, w1, w2, zl) + vsig * qv[u]);
                if (pb + u < p1) {
                    r[pb + u] = rv;
                    alpha += (double)(vsc * qv[u]) * (double)rv;
                }
            }
            }
        }
    }
    if (alpha_base != nullptr) {
        alpha = block_sum(alpha, red);
        if (threadIdx.x == 0) atomicAdd(alpha_base, alpha);
    }
}

// d <= 2 gather, thread per 4 consecutive sorted points (coalesced q / frac / cell loads and r
// stores; the z stencil loads of neighbouring points hit the same lines):
//   r_p = sum_l w_l(p) z[cell(p) - 1 + l] + sigma^2 s_j Q~_j[p],   alpha += s_j Q~_j[p] r_p
// Same per-point arithmetic as gather_kernel<V, 1>; points past n get r = 0.
template <typename V>
__device__ __forceinline__ void ld4(const V* __restrict__ p, V o[4]) {
    if constexpr (sizeof(V) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
        const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
        o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    }
}
template <typename V>
__device__ __forceinline__ void st4(V* __restrict__ p, const V o[4]) {
    if constexpr (sizeof(V) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
        reinterpret_cast<double2*>(p)[0] = make_double2(o[0], o[1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(o[2], o[3]);
    }
}

template <typename V, int D>
__global__ void __launch_bounds__(256) gather_pts1_kernel(GridDev g, int64_t n, int64_t ngroups,
                                                          const int* __restrict__ pcell, const V* __restrict__ f0,
                                                          const V* __restrict__ f1, const double* __restrict__ z,
                                                          const V* __restrict__ qbase, StepRef ref, double sigma2,
                                                          V* __restrict__ r, double* __restrict__ alpha_base,
                                                          RcStream rs, int nstream) {
    pdl_wait();
    LOVE_TRACE(kTrGather, step_j(ref));
    // the first nstream CTAs stream the cache column (they start first and overlap the gather)
    if ((int)blockIdx.x < nstream) {
        stream_rc_column(rs, blockIdx.x * blockDim.x + threadIdx.x, nstream * blockDim.x);
        return;
    }
    using A = typename AccT<V, D>::type;
    __shared__ double red[32];
    if (step_done(ref)) return;
    const int j = step_j(ref);
    const V* __restrict__ q = qbase + j * ref.ld;
    const double sc = ref.scale[j];
    const A vsc = (A)sc, vsig = (A)(sigma2 * sc);
    double alpha = 0.0;
    const int64_t t = (blockIdx.x - nstream) * (int64_t)blockDim.x + threadIdx.x;
    if (t < ngroups) {
        const int64_t p0 = t * 4;
        V qv[4], fa[4], fb[4], rv[4];
        ld4<V>(q + p0, qv);
        ld4<V>(f0 + p0, fa);
        if (D > 1) ld4<V>(f1 + p0, fb);
        const int4 cl = *reinterpret_cast<const int4*>(pcell + p0);
        const int cells[4] = {cl.x, cl.y, cl.z, cl.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            rv[u] = V(0);
            if (p0 + u < n) {
                A zl[Slots<D>::value], w0[4], w1[4];
                load_stencil<A, D>(g, z, D == 1 ? cells[u] - 1 : stencil_base<D>(g, cells[u]), zl);
                keys4<A>((A)fa[u], w0);
                if (D > 1) keys4<A>((A)fb[u], w1);
                const A qa = (A)qv[u];
                rv[u] = (V)(stencil_dot<A, D>(w0, w1, w1, zl) + vsig * qa);
                alpha += (double)(vsc * qa) * (double)rv[u];
            }
        }
        st4<V>(r + p0, rv);
    }
    if (alpha_base != nullptr) {
        alpha = block_sum(alpha, red);
        if (threadIdx.x == 0) atomicAdd(alpha_base, alpha);
    }
}

// d = 1: per-cell stencil moments, TPC (= 2) lanes per cell, already scaled by q_j's column scale:
//   Mc[l][c + 2] = s_j * sum_{p in cell c} w_l(p) Q~_j[p]      (l = 0..3, rows of length m + 4)
// so that (W q_j)[i] = Mc[0][i+3] + Mc[1][i+2] + Mc[2][i+1] + Mc[3][i]  (no atomics, fixed order)
template <typename V, int TPC>
__global__ void __launch_bounds__(256) moments_cell1_kernel(int m, const int* __restrict__ cell_start,
                                                            const V* __restrict__ f0, const V* __restrict__ qbase,
                                                            StepRef ref, double* __restrict__ Mc) {
    pdl_wait();
    LOVE_TRACE(kTrMoments, step_j(ref));
    // TPC lanes per cell (aligned lane groups): lane `sub` takes points p0 + sub, p0 + sub + TPC, ...
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = gt / TPC, sub = gt % TPC;
    if (step_done(ref)) return;
    const bool live = c < m;
    const int j = step_j(ref);
    const V* __restrict__ q = qbase + j * ref.ld;
    const int p0 = live ? cell_start[c] : 0, p1 = live ? cell_start[c + 1] : 0;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int B = kBatch / TPC > 2 ? kBatch / TPC : 2;
    for (int pb = p0 + sub; pb < p1; pb += B * TPC) {
        double qv[B], fa[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int p = pb + u * TPC;
            const bool in = p < p1;
            qv[u] = in ? (double)q[p] : 0.0;
            fa[u] = in ? (double)f0[p] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            double w[4];
            keys4<double>(fa[u], w);
#pragma unroll
            for (int l = 0; l < 4; ++l) acc[l] += w[l] * qv[u];
        }
    }
#pragma unroll
    for (int o = 1; o < TPC; o <<= 1)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], o);
    if (!live || sub != 0) return;
    const double sc = ref.scale[j];
    const int ld = m + 4;
#pragma unroll
    for (int l = 0; l < 4; ++l) Mc[l * ld + c + 2] = acc[l] * sc;
}

__global__ void __launch_bounds__(256) nodepass_cell1_kernel(int m, const double* __restrict__ Mc, StepRef ref,
                                                             double* __restrict__ u) {
    pdl_wait();
    LOVE_TRACE(kTrNodepass, step_j(ref));
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || step_done(ref)) return;
    const int ld = m + 4;
    u[i] = Mc[i + 3] + Mc[ld + i + 2] + Mc[2 * ld + i + 1] + Mc[3 * ld + i];
}

template <typename V>
__global__ void permute_kernel(const int* __restrict__ perm, int64_t n, const V* __restrict__ in,
                               V* __restrict__ out, int to_sorted) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        if (to_sorted) out[p] = in[perm[p]];
        else out[perm[p]] = in[p];
    }
}

template <typename A, typename B>
__global__ void convert_kernel(const A* __restrict__ in, B* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (B)in[i];
}

// threads per CTA of the 3-D item kernels (LOVE_ITEM_BLOCK3 = 64 .. 256, a multiple of 32).
// At 128 registers a CTA of 128 threads is retired (and its slot refilled) when its 4 warps are
// done, not 8: the items' uneven lengths idle fewer warp slots.  Measured (cfg4, in-graph):
// 256 threads moments 25.7 / gather 33.3 us, 192: 26.1 / 36.8, 128: 23.1 / 31.4, 64: 22.7 / 31.5;
// cfg4 28.02 -> 27.60 ms at 128.
int item_block3() {
    static const int v = [] {
        const char* e = std::getenv("LOVE_ITEM_BLOCK3");
        const int b = e ? std::atoi(e) : 128;
        return b >= 64 && b <= 256 && b % 32 == 0 ? b : 128;
    }();
    return v;
}

}  // namespace

void launch_nodepass(const Cache& c, StepRef ref, double* u, cudaStream_t s) {
    const int gm = (int)ceil_div(c.g.m_total, 256);
    const double* M = (const double*)c.M;
    switch (c.g.d) {
        case 1: LOVE_LAUNCH((nodepass_kernel<1>), gm, 256, 0, s, c.g, c.n_items, c.cell_item_start, M, ref, u); break;
        case 2: LOVE_LAUNCH((nodepass_kernel<2>), gm, 256, 0, s, c.g, c.n_items, c.cell_item_start, M, ref, u); break;
        default: LOVE_LAUNCH((nodepass_kernel<3>), gm, 256, 0, s, c.g, c.n_items, c.cell_item_start, M, ref, u); break;
    }
}

template <typename V>
void launch_scatter(const Cache& c, const V* q, StepRef ref, double* u, cudaStream_t s, bool moments_only) {
    if (c.additive) {
        add_scatter<V>(c, q, ref, u, s);
        return;
    }
    if (c.g.d == 1 && c.Mc != nullptr) {
        const int m = c.g.m_total;
        LOVE_LAUNCH((moments_cell1_kernel<V, 2>), (int)ceil_div(2 * (int64_t)m, 256), 256, 0, s, m, c.cell_start,
                    (const V*)c.frac[0], q, ref, (double*)c.Mc);
        if (!moments_only)
            LOVE_LAUNCH(nodepass_cell1_kernel, (int)ceil_div(m, 256), 256, 0, s, m, (const double*)c.Mc, ref, u);
        return;
    }
    const int64_t ni = c.n_items;
    const int gi = (int)std::max<int64_t>(1, ceil_div(ni, 256));
    const V* f0 = (const V*)c.frac[0];
    const V* f1 = (const V*)c.frac[1];
    const V* f2 = (const V*)c.frac[2];
    double* M = (double*)c.M;
    const int m = c.g.m_total;
    if (c.g.d >= 2 && c.pullT != nullptr) {
        if (c.g.d == 2) {
            if (ni)
                LOVE_LAUNCH(moments2_tpc_kernel<V>, (int)ceil_div(2 * ni, 256), 256, 0, s, ni, c.item_start, f0, f1, q,
                            ref, M);
            constexpr int SG2 = LOVE_PULL2_SG;
            LOVE_LAUNCH((pull_last_kernel<2, double, SG2>), (int)ceil_div((int64_t)m * (4 / SG2), 256), 256, 0, s,
                        c.g, ni, c.cell_item_start, (const double*)M, ref, (double*)c.pullT);
            LOVE_LAUNCH(pull_first_kernel, (int)ceil_div(m, 256), 256, 0, s, c.g, (const double*)c.pullT, ref, u);
        } else {
            // the 3-D moments are stored in their accumulation type (fp32 in LOVE_FP32 mode)
            using MT = typename AccT<V, 3>::type;
            MT* Mf = (MT*)c.M;
            if (ni) {
                const int tb = item_block3();
                LOVE_LAUNCH((moments_kernel<V, 3, MT>), (int)ceil_div(ni, tb), tb, 0, s, ni, c.item_start, f0, f1, f2, q,
                            ref, Mf);
            }
            constexpr int SG = LOVE_PULL3_SG;
            // fp32 moments: the per-slot last-axis sums T are stored in fp32 too (half the bytes of
            // the T round trip; u is summed in fp64 by the next pull); LOVE_PULL_T64=1: fp64 T
            static const bool t64 = std::getenv("LOVE_PULL_T64") != nullptr;
            const bool tf32 = std::is_same<MT, float>::value && !t64;
            if (tf32)
                LOVE_LAUNCH((pull_last_kernel<3, MT, SG, float>), (int)ceil_div((int64_t)m * (16 / SG), 256), 256, 0, s,
                            c.g, ni, c.cell_item_start, (const MT*)Mf, ref, (float*)c.pullT);
            else
                LOVE_LAUNCH((pull_last_kernel<3, MT, SG>), (int)ceil_div((int64_t)m * (16 / SG), 256), 256, 0, s, c.g,
                            ni, c.cell_item_start, (const MT*)Mf, ref, (double*)c.pullT);
            static const bool split = std::getenv("LOVE_PULL_MF") != nullptr && std::atoi(std::getenv("LOVE_PULL_MF")) == 0;
            if (split && !tf32) {
                LOVE_LAUNCH(pull_mid_kernel, (int)ceil_div(4 * (int64_t)m, 256), 256, 0, s, c.g,
                            (const double*)c.pullT, ref, (double*)c.pullV);
                LOVE_LAUNCH(pull_first_kernel, (int)ceil_div(m, 256), 256, 0, s, c.g, (const double*)c.pullV, ref, u);
            } else if (moments_only && tf32) {
                // fuse_pull3: the first K_UU axis product forms u from T itself (launch_kuu(..., pull3))
            } else {
                if (tf32)
                    LOVE_LAUNCH(pull_mid_first_kernel<float>, (int)ceil_div(m, 256), 256, 0, s, c.g,
                                (const float*)c.pullT, ref, u);
                else
                    LOVE_LAUNCH(pull_mid_first_kernel<double>, (int)ceil_div(m, 256), 256, 0, s, c.g,
                                (const double*)c.pullT, ref, u);
            }
        }
        return;
    }
    if (ni) {
        switch (c.g.d) {
            case 1: LOVE_LAUNCH((moments_kernel<V, 1, double>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, ref, M); break;
            case 2: LOVE_LAUNCH((moments_kernel<V, 2, double>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, ref, M); break;
            default: LOVE_LAUNCH((moments_kernel<V, 3, double>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, ref, M); break;
        }
    }
    launch_nodepass(c, ref, u, s);
}

template <typename V>
void launch_gather(const Cache& c, const double* z, const V* q, StepRef ref, V* r, double* alpha_base,
                   cudaStream_t s, const RcStream* rsp) {
    if (c.additive) {
        add_gather<V>(c, z, q, ref, r, alpha_base, s, rsp);
        return;
    }
    RcStream rs{};
    int extra = 0;
    if (rsp != nullptr) {
        rs = *rsp;
        extra = (int)std::min<int64_t>(ceil_div(rs.m, 256), 148 * 2);
    }
    if (c.g.d <= 2 && c.pcell != nullptr) {
        const int64_t ng = c.ldq / 4;
        const int gq = (int)ceil_div(ng, 256);
        if (gq + extra > 0) {
            if (c.g.d == 1)
                LOVE_LAUNCH((gather_pts1_kernel<V, 1>), gq + extra, 256, 0, s, c.g, c.n, ng, (const int*)c.pcell,
                            (const V*)c.frac[0], (const V*)c.frac[0], z, q, ref, c.sigma2, r, alpha_base, rs, extra);
            else
                LOVE_LAUNCH((gather_pts1_kernel<V, 2>), gq + extra, 256, 0, s, c.g, c.n, ng, (const int*)c.pcell,
                            (const V*)c.frac[0], (const V*)c.frac[1], z, q, ref, c.sigma2, r, alpha_base, rs, extra);
        }
        return;
    }
    const int64_t ni = c.n_items;
    const int gi = (int)ceil_div(ni, 256);
    if (gi + extra == 0) return;
    const V* f0 = (const V*)c.frac[0];
    const V* f1 = (const V*)c.frac[1];
    const V* f2 = (const V*)c.frac[2];
#define LOVE_GATHER(DD)                                                                                       \
    LOVE_LAUNCH((gather_kernel<V, DD>), gi + extra, 256, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1, f2, z, \
                q, ref, c.sigma2, r, alpha_base, rs, gi)
    switch (c.g.d) {
        case 1: LOVE_GATHER(1); break;
        case 2: LOVE_GATHER(2); break;
        default: {
            const int tb = item_block3();
            const int g3 = (int)ceil_div(ni, tb);
            const int ex3 = rsp != nullptr ? (int)std::min<int64_t>(ceil_div(rs.m, tb), 148 * 2 * (256 / tb)) : 0;
            LOVE_LAUNCH((gather_kernel<V, 3>), g3 + ex3, tb, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1, f2, z, q,
                        ref, c.sigma2, r, alpha_base, rs, g3);
            break;
        }
    }
#undef LOVE_GATHER
}

template <typename V>
void launch_permute(const Cache& c, const V* in, V* out, bool to_sorted, cudaStream_t s) {
    if (c.n == 0) return;
    const int gb = (int)std::min<int64_t>(ceil_div(c.n, 256), 148 * 32);
    LOVE_LAUNCH(permute_kernel<V>, gb, 256, 0, s, c.perm, c.n, in, out, to_sorted ? 1 : 0);
}

template <typename A, typename B>
void launch_convert(const A* in, B* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    LOVE_LAUNCH((convert_kernel<A, B>), (int)std::min<int64_t>(ceil_div(n, 256), 148 * 16), 256, 0, s, in, out, n);
}

template void launch_convert<float, double>(const float*, double*, int64_t, cudaStream_t);
template void launch_convert<double, float>(const double*, float*, int64_t, cudaStream_t);
template void launch_scatter<float>(const Cache&, const float*, StepRef, double*, cudaStream_t, bool);
template void launch_scatter<double>(const Cache&, const double*, StepRef, double*, cudaStream_t, bool);
template void launch_gather<float>(const Cache&, const double*, const float*, StepRef, float*, double*,
                                   cudaStream_t, const RcStream*);
template void launch_gather<double>(const Cache&, const double*, const double*, StepRef, double*, double*,
                                    cudaStream_t, const RcStream*);
template void launch_permute<float>(const Cache&, const float*, float*, bool, cudaStream_t);
template void launch_permute<double>(const Cache&, const double*, double*, bool, cudaStream_t);

}  // namespace love
