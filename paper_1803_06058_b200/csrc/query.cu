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

__device__ __forceinline__ Stencil make_stencil(const GridDev& g, const double* x) {
    Stencil s;
    s.ok = true;
    s.base = 0;
    for (int d = 0; d < 3; ++d) {
        s.j[d] = 0;
        for (int e = 0; e < 4; ++e) s.w[d][e] = 0.0;
    }
    for (int d = 0; d < g.d; ++d) {
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
__device__ __forceinline__ double prior_ski(const GridDev& g, const double* cols64, double s2,
                                            const Stencil& A, const Stencil& B) {
    double p = s2;
    int off = 0;
    for (int d = 0; d < g.d; ++d) {
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

template <typename V, int D>
__global__ void __launch_bounds__(256) predict_kernel(GridDev g, const double* __restrict__ cols64, double s2,
                                                      double l0, double l1, double l2, int prior_mode,
                                                      const V* __restrict__ Rc, int k_pad,
                                                      const double* __restrict__ amean,
                                                      const double* __restrict__ Xa,
                                                      const double* __restrict__ Xb, int64_t t,
                                                      V* __restrict__ out, V* __restrict__ mean_out,
                                                      unsigned long long* __restrict__ counters) {
    constexpr int W = QV<V>::W;
    using VT = typename QV<V>::T;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nchunks = k_pad / W;
    const bool covar = Xb != nullptr;
    for (int64_t qi = warp; qi < t; qi += nwarps) {
        const Stencil A = make_stencil(g, Xa + qi * D);
        const Stencil B = covar ? make_stencil(g, Xb + qi * D) : A;
        if (!(A.ok && B.ok)) {
            if (lane == 0) {
                out[qi] = (V)NAN;
                if (mean_out) mean_out[qi] = (V)NAN;
                atomicAdd(&counters[1], 1ull);
            }
            continue;
        }
        double dot = 0.0;
        for (int c0 = 0; c0 < nchunks; c0 += 32) {
            const int ch = c0 + lane;
            if (ch >= nchunks) break;
            double ra[W], rb[W];
#pragma unroll
            for (int e = 0; e < W; ++e) ra[e] = rb[e] = 0.0;
#pragma unroll
            for (int pass = 0; pass < 2; ++pass) {
                if (pass == 1 && !covar) break;
                const Stencil& S = pass == 0 ? A : B;
                double* acc = pass == 0 ? ra : rb;
#pragma unroll
                for (int a = 0; a < 4; ++a) {
#pragma unroll
                    for (int b = 0; b < (D > 1 ? 4 : 1); ++b) {
#pragma unroll
                        for (int cc = 0; cc < (D > 2 ? 4 : 1); ++cc) {
                            int node = S.base;
                            double w = S.w[0][a];
                            if (D == 1) node += a;
                            if (D == 2) { node += a * g.stride[0] + b; w *= S.w[1][b]; }
                            if (D == 3) {
                                node += a * g.stride[0] + b * g.stride[1] + cc;
                                w *= S.w[1][b] * S.w[2][cc];
                            }
                            const VT v = *reinterpret_cast<const VT*>(Rc + (int64_t)node * k_pad + ch * W);
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
            if (!covar)
                for (int e = 0; e < W; ++e) rb[e] = ra[e];
#pragma unroll
            for (int e = 0; e < W; ++e) dot += ra[e] * rb[e];
        }
        dot = warp_sum(dot);
        if (lane == 0) {
            double prior;
            if (prior_mode == LOVE_PRIOR_EXACT) {
                const double ls[3] = {l0, l1, l2};
                double r2 = 0.0;
                for (int d = 0; d < D; ++d) {
                    const double df = Xa[qi * D + d] - (covar ? Xb[qi * D + d] : Xa[qi * D + d]);
                    r2 += df * df / (ls[d] * ls[d]);
                }
                prior = s2 * exp(-0.5 * r2);
            } else {
                prior = prior_ski(g, cols64, s2, A, B);
            }
            const double v = prior - dot;
            out[qi] = (V)v;
            if (!covar && v < 0.0) atomicAdd(&counters[0], 1ull);
            if (mean_out) {
                double mu = 0.0;
                for (int a = 0; a < 4; ++a)
                    for (int b = 0; b < (D > 1 ? 4 : 1); ++b)
                        for (int cc = 0; cc < (D > 2 ? 4 : 1); ++cc) {
                            int node = A.base;
                            double w = A.w[0][a];
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
}

}  // namespace

template <typename V>
void launch_predict(const Cache& c, const double* Xa, const double* Xb, int64_t t, V* out, V* mean_out,
                    cudaStream_t s) {
    if (t <= 0) return;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(t, 8), 148 * 16));
    const double* L = c.rbf.lengthscale;
    switch (c.g.d) {
        case 1:
            LOVE_LAUNCH((predict_kernel<V, 1>), blocks, 256, 0, s, c.g, c.cols64, c.rbf.outputscale, L[0], L[1],
                        L[2], c.prior, (const V*)c.Rc, c.k_pad, (const double*)c.a, Xa, Xb, t, out, mean_out,
                        c.counters);
            break;
        case 2:
            LOVE_LAUNCH((predict_kernel<V, 2>), blocks, 256, 0, s, c.g, c.cols64, c.rbf.outputscale, L[0], L[1],
                        L[2], c.prior, (const V*)c.Rc, c.k_pad, (const double*)c.a, Xa, Xb, t, out, mean_out,
                        c.counters);
            break;
        default:
            LOVE_LAUNCH((predict_kernel<V, 3>), blocks, 256, 0, s, c.g, c.cols64, c.rbf.outputscale, L[0], L[1],
                        L[2], c.prior, (const V*)c.Rc, c.k_pad, (const double*)c.a, Xa, Xb, t, out, mean_out,
                        c.counters);
            break;
    }
}

template void launch_predict<float>(const Cache&, const double*, const double*, int64_t, float*, float*,
                                    cudaStream_t);
template void launch_predict<double>(const Cache&, const double*, const double*, int64_t, double*, double*,
                                     cudaStream_t);

}  // namespace love
