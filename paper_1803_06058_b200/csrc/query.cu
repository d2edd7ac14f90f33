// query.cu -- O(k) predictive (co)variance and mean queries (Eq. 10; Alg. 1
// P:401-403; Eq. 6).
//
// One warp per query.  Interpolation (cell, Keys weights) and the prior are computed in
// fp64 (reading A21: the cancellation prior - ||Rc^T w||^2 needs fp64 weights); lanes own
// 16-byte chunks of the k-vector r = sum_l w_l Rc[node_l, :] and accumulate in fp64.  For
// d = 1 the 4 stencil rows of Rc are contiguous (4 * k_pad values), for d = 3 they are 16
// runs of 4 rows.
#include <cuda_runtime.h>

#include <cmath>

#include "love_internal.h"

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

}  // namespace

template <typename V>
void launch_predict(const Cache& c, const double* Xa, const double* Xb, int64_t t, V* out, V* mean_out,
                    cudaStream_t s) {
    if (t <= 0) return;
    ProfScope ps(LOVE_PROF_QUERY, s);
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
