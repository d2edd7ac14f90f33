// additive.cu -- LOVE for additive kernel compositions (Eq. 16).
//
//   k(x, x') = sum_e w^(e)_x^T K^(e)_UU w^(e)_x'  =  [w^(1); ..; w^(d)]^T diag(K^(1), .., K^(d)) [..]
//
// Algorithm 1 runs on the block forms: the interpolation vector of a point stacks
// the 1-D cubic stencils of its d components (4 nonzeros each, "O(d)-sparse"), and
// K_UU is block diagonal with one Toeplitz block per component ("O(d m log m)"; here a
// dense Toeplitz product per block from shared memory, m_e <= 1024).  The Lanczos driver,
// the streamed cache and the queries are the grid code's; this file supplies the
// structure-specific operators:
//   scatter  u = W q       : per component, points counting-sorted by their component cell;
//                            one warp per cell sums its 4 stencil moments (fixed order, no
//                            atomics), then a node pass u[off_e + i] = sum_s M_s[off_e + i+1-s]
//   K_UU u                 : one CTA per component
//   gather   r = W^T z + s2 q, alpha : one thread per point, 4d z values
//   queries                : G lanes per query over the k-vector, 4d rows of Rc
// Training points keep their original order (the cache's perm is the identity).
#include <cuda_runtime.h>

#include <cmath>

#include "love_internal.h"

namespace love {

namespace {

__device__ __forceinline__ int comp_of(const AddDev& a, int g) {
    int e = 0;
    while (e + 1 < a.d && g >= a.off[e + 1]) ++e;
    return e;
}

// cells and fractions per component (fp64 floor, reading A3; range rule A4)
template <typename V>
__global__ void add_interp_kernel(AddDev a, const double* __restrict__ X, int64_t n, int* __restrict__ acell,
                                  V* __restrict__ afrac, int* __restrict__ flag) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        for (int e = 0; e < a.d; ++e) {
            const double sc = (X[p * a.d + e] - a.lo[e]) / a.h[e];
            const double jf = floor(sc);
            const bool ok = jf >= 1.0 && jf <= (double)(a.m[e] - 3);
            acell[e * n + p] = ok ? (int)jf : 1;
            afrac[e * n + p] = (V)(ok ? sc - jf : 0.0);
            if (!ok) atomicOr(flag, 1);
        }
    }
}

// c_e[i] = exp(-(i h_e)^2 / (2 l_e^2)) at cols[off_e + i]  (reading A6)
__global__ void add_columns_kernel(AddDev a, double* __restrict__ cols) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < a.off[a.d]; g += gridDim.x * blockDim.x) {
        const int e = comp_of(a, g);
        const double r = (double)(g - a.off[e]) * a.h[e];
        cols[g] = exp(-(r * r) / (2.0 * a.ls[e] * a.ls[e]));
    }
}

__global__ void iota_kernel(int* __restrict__ p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = (int)i;
}

// one warp per component cell (a component cell holds ~n / m_e points): lanes stride over the
// cell's points in fixed order, four fp64 partial sums per lane, then a warp reduction
template <typename V>
__global__ void __launch_bounds__(256) add_moments_kernel(AddDev a, int64_t n, const int* __restrict__ aperm,
                                                          const int* __restrict__ astart, const V* __restrict__ afrac,
                                                          const V* __restrict__ qbase, StepRef ref,
                                                          double* __restrict__ Mc) {
    pdl_wait();
    const int M = a.off[a.d];
    const int g = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (g >= M || step_done(ref)) return;
    const int j = step_j(ref);
    const V* __restrict__ q = qbase + j * ref.ld;
    const int e = comp_of(a, g), c = g - a.off[e];
    const int* __restrict__ st = astart + a.off[e] + e;
    const int* __restrict__ pe = aperm + (int64_t)e * n;
    const V* __restrict__ fe = afrac + (int64_t)e * n;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int i1 = st[c + 1];
    for (int i = st[c] + lane; i < i1; i += 32) {
        const int p = pe[i];
        double w[4];
        keys4<double>((double)fe[p], w);
        const double qv = (double)q[p];
#pragma unroll
        for (int s = 0; s < 4; ++s) acc[s] += w[s] * qv;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) acc[s] = warp_sum(acc[s]);
    if (lane != 0) return;
    const double sc = ref.scale[j];
#pragma unroll
    for (int s = 0; s < 4; ++s) Mc[(int64_t)s * M + g] = acc[s] * sc;
}

__global__ void __launch_bounds__(256) add_nodepass_kernel(AddDev a, const double* __restrict__ Mc, StepRef ref,
                                                           double* __restrict__ u) {
    pdl_wait();
    const int M = a.off[a.d];
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= M || step_done(ref)) return;
    const int e = comp_of(a, g), i = g - a.off[e];
    double sum = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {           // slot s of cell c = i + 1 - s lands on node i
        const int c = i + 1 - s;
        if (c >= 0 && c < a.m[e]) sum += Mc[(int64_t)s * M + a.off[e] + c];
    }
    u[g] = sum;
}

// block e of K_UU: z_e = s2_e T(c_e) u_e, one CTA per component (m_e <= 1024)
__global__ void __launch_bounds__(256) add_kuu_kernel(AddDev a, const double* __restrict__ cols,
                                                      const double* __restrict__ u, double* __restrict__ z) {
    pdl_wait();
    __shared__ double us[1024], cs[1024];
    const int e = blockIdx.x;
    const int m = a.m[e], off = a.off[e];
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        us[i] = u[off + i];
        cs[i] = cols[off + i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        double acc0 = 0.0, acc1 = 0.0;
        int jj = 0;
        for (; jj + 1 < m; jj += 2) {
            acc0 += cs[abs(i - jj)] * us[jj];
            acc1 += cs[abs(i - jj - 1)] * us[jj + 1];
        }
        if (jj < m) acc0 += cs[abs(i - jj)] * us[jj];
        z[off + i] = a.s2[e] * (acc0 + acc1);
    }
}

template <typename V>
__global__ void __launch_bounds__(256) add_gather_kernel(AddDev a, int64_t n, const int* __restrict__ acell,
                                                         const V* __restrict__ afrac, const double* __restrict__ z,
                                                         const V* __restrict__ qbase, StepRef ref, double sigma2,
                                                         V* __restrict__ r, double* __restrict__ alpha_base,
                                                         RcStream rs, int ngather) {
    pdl_wait();
    if ((int)blockIdx.x >= ngather) {
        stream_rc_column(rs, (blockIdx.x - ngather) * blockDim.x + threadIdx.x, (gridDim.x - ngather) * blockDim.x);
        return;
    }
    __shared__ double red[32];
    if (step_done(ref)) return;
    const int j = step_j(ref);
    const V* __restrict__ q = qbase + j * ref.ld;
    const double sc = ref.scale[j];
    double alpha = 0.0;
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p < n) {
        double acc = 0.0;
        for (int e = 0; e < a.d; ++e) {
            const int c = acell[e * n + p];
            double w[4];
            keys4<double>((double)afrac[e * n + p], w);
            const double* ze = z + a.off[e] + c - 1;
            acc += w[0] * ze[0] + w[1] * ze[1] + w[2] * ze[2] + w[3] * ze[3];
        }
        const double qv = (double)q[p];
        const V rv = (V)(acc + sigma2 * sc * qv);
        r[p] = rv;
        alpha = (sc * qv) * (double)rv;
    }
    if (alpha_base != nullptr) {
        alpha = block_sum(alpha, red);
        if (threadIdx.x == 0) atomicAdd(alpha_base, alpha);
    }
}

template <typename V> struct AV;
template <> struct AV<float> { using T = float4; static constexpr int W = 4; };
template <> struct AV<double> { using T = double2; static constexpr int W = 2; };

// 1-D stencil of component e for a query coordinate (fp64, reading A21); false if outside
__device__ __forceinline__ bool add_stencil(const AddDev& a, int e, double x, int& cell, double w[4]) {
    const double sc = (x - a.lo[e]) / a.h[e];
    const double jf = floor(sc);
    const bool ok = jf >= 1.0 && jf <= (double)(a.m[e] - 3);
    cell = ok ? (int)jf : 1;
    keys4<double>(ok ? sc - jf : 0.0, w);
    return ok;
}

// variances (Xb == nullptr) or pair covariances: prior - (Rc^T w_a) . (Rc^T w_b)   (Eq. 10)
template <typename V, int G>
__global__ void __launch_bounds__(256) add_predict_kernel(AddDev a, const double* __restrict__ cols, int prior_mode,
                                                          const V* __restrict__ Rc, int k_pad,
                                                          const double* __restrict__ amean,
                                                          const double* __restrict__ Xa, const double* __restrict__ Xb,
                                                          int64_t t, V* __restrict__ out, V* __restrict__ mean_out,
                                                          unsigned long long* __restrict__ counters) {
    constexpr int W = AV<V>::W;
    using VT = typename AV<V>::T;
    constexpr int QPW = 32 / G;
    const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nch = k_pad / W;
    const bool covar = Xb != nullptr;
    const int d = a.d;
    for (int64_t base = warp * QPW; base < t; base += nwarps * QPW) {
        const int64_t qi = base + sub;
        const bool active = qi < t;
        const int64_t qq = active ? qi : base;
        const double* xa = Xa + qq * d;
        const double* xb = covar ? Xb + qq * d : xa;
        bool ok = active;
        double dot = 0.0;
        for (int ch = gl; ch < nch; ch += G) {
            double ra[W], rb[W];
#pragma unroll
            for (int e2 = 0; e2 < W; ++e2) { ra[e2] = 0.0; rb[e2] = 0.0; }
            for (int e = 0; e < d; ++e) {
                int ca, cb;
                double wa[4], wb[4];
                ok = add_stencil(a, e, xa[e], ca, wa) && ok;
                ok = add_stencil(a, e, xb[e], cb, wb) && ok;
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const VT va = __ldg(reinterpret_cast<const VT*>(Rc + (int64_t)(a.off[e] + ca - 1 + s) * k_pad + ch * W));
                    const VT vb = covar ? __ldg(reinterpret_cast<const VT*>(Rc + (int64_t)(a.off[e] + cb - 1 + s) * k_pad + ch * W)) : va;
                    if constexpr (W == 4) {
                        ra[0] += wa[s] * (double)va.x; ra[1] += wa[s] * (double)va.y;
                        ra[2] += wa[s] * (double)va.z; ra[3] += wa[s] * (double)va.w;
                        rb[0] += wb[s] * (double)vb.x; rb[1] += wb[s] * (double)vb.y;
                        rb[2] += wb[s] * (double)vb.z; rb[3] += wb[s] * (double)vb.w;
                    } else {
                        ra[0] += wa[s] * (double)va.x; ra[1] += wa[s] * (double)va.y;
                        rb[0] += wb[s] * (double)vb.x; rb[1] += wb[s] * (double)vb.y;
                    }
                }
            }
#pragma unroll
            for (int e2 = 0; e2 < W; ++e2) dot += ra[e2] * rb[e2];
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (gl != 0 || !active) continue;
        // the stencils again on the writing lane (cheap; ok also for nch < G lanes)
        double prior = 0.0, mu = 0.0;
        bool okw = true;
        for (int e = 0; e < d; ++e) {
            int ca, cb;
            double wa[4], wb[4];
            okw = add_stencil(a, e, xa[e], ca, wa) && okw;
            okw = add_stencil(a, e, xb[e], cb, wb) && okw;
            if (prior_mode == LOVE_PRIOR_EXACT) {
                const double df = xa[e] - xb[e];
                prior += a.s2[e] * exp(-0.5 * df * df / (a.ls[e] * a.ls[e]));
            } else {
                double acc = 0.0;
#pragma unroll
                for (int s1 = 0; s1 < 4; ++s1)
#pragma unroll
                    for (int s2 = 0; s2 < 4; ++s2) {
                        const int dist = abs((ca + s1) - (cb + s2));
                        acc += wa[s1] * wb[s2] * (covar ? cols[a.off[e] + dist] : a.c4[e][dist]);
                    }
                prior += a.s2[e] * acc;
            }
            if (mean_out) {
#pragma unroll
                for (int s = 0; s < 4; ++s) mu += wa[s] * amean[a.off[e] + ca - 1 + s];
            }
        }
        if (!okw) {
            out[qi] = (V)NAN;
            if (mean_out) mean_out[qi] = (V)NAN;
            atomicAdd(&counters[1], 1ull);
            continue;
        }
        const double v = prior - dot;
        out[qi] = (V)v;
        if (!covar && v < 0.0) atomicAdd(&counters[0], 1ull);
        if (mean_out) mean_out[qi] = (V)mu;
    }
}

}  // namespace

void additive_setup(Cache& c, const double* X, const double* y, int* range_flag, cudaStream_t s) {
    const AddDev& a = c.ad;
    const int64_t n = c.n;
    const int M = a.off[a.d];
    const size_t vs = c.vsize;
    c.acell = (int*)dalloc(c, sizeof(int) * (size_t)a.d * std::max<int64_t>(n, 1), s);
    c.afrac = dalloc(c, vs * (size_t)a.d * std::max<int64_t>(n, 1), s);
    c.aperm = (int*)dalloc(c, sizeof(int) * (size_t)a.d * std::max<int64_t>(n, 1), s);
    c.astart = (int*)dalloc(c, sizeof(int) * (size_t)(M + a.d), s);
    c.aMc = dalloc(c, sizeof(double) * 4 * (size_t)M, s);
    c.perm = (int*)dalloc(c, sizeof(int) * std::max<int64_t>(n, 1), s);
    c.cols64 = (double*)dalloc(c, sizeof(double) * M, s);
    const int gb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 16));
    if (n > 0) {
        if (c.precision == LOVE_FP64)
            LOVE_LAUNCH(add_interp_kernel<double>, gb, 256, 0, s, a, X, n, c.acell, (double*)c.afrac, range_flag);
        else
            LOVE_LAUNCH(add_interp_kernel<float>, gb, 256, 0, s, a, X, n, c.acell, (float*)c.afrac, range_flag);
        for (int e = 0; e < a.d; ++e)
            counting_sort_keys(c.acell + (int64_t)e * n, n, a.m[e], c.astart + a.off[e] + e,
                               c.aperm + (int64_t)e * n, s);
        LOVE_LAUNCH(iota_kernel, gb, 256, 0, s, c.perm, n);
    }
    LOVE_LAUNCH(add_columns_kernel, (int)ceil_div(M, 256), 256, 0, s, a, c.cols64);
}

template <typename V>
void add_scatter(const Cache& c, const V* q, StepRef ref, double* u, cudaStream_t s) {
    const int M = c.ad.off[c.ad.d];
    LOVE_LAUNCH(add_moments_kernel<V>, (int)ceil_div((int64_t)M * 32, 256), 256, 0, s, c.ad, c.n, c.aperm, c.astart,
                (const V*)c.afrac, q, ref, (double*)c.aMc);
    LOVE_LAUNCH(add_nodepass_kernel, (int)ceil_div(M, 256), 256, 0, s, c.ad, (const double*)c.aMc, ref, u);
}

void add_kuu(const Cache& c, const double* u, double* z, cudaStream_t s) {
    LOVE_LAUNCH(add_kuu_kernel, c.ad.d, 256, 0, s, c.ad, (const double*)c.cols64, u, z);
}

template <typename V>
void add_gather(const Cache& c, const double* z, const V* q, StepRef ref, V* r, double* alpha_base, cudaStream_t s,
                const RcStream* rsp) {
    RcStream rs{};
    int extra = 0;
    if (rsp != nullptr) {
        rs = *rsp;
        extra = (int)std::min<int64_t>(ceil_div(rs.m, 256), 148 * 2);
    }
    const int gp = (int)ceil_div(c.n, 256);
    if (gp + extra == 0) return;
    LOVE_LAUNCH(add_gather_kernel<V>, gp + extra, 256, 0, s, c.ad, c.n, c.acell, (const V*)c.afrac, z, q, ref,
                c.sigma2, r, alpha_base, rs, gp);
}

template <typename V>
void add_predict(const Cache& c, const double* Xa, const double* Xb, int64_t t, V* out, V* mean_out,
                 cudaStream_t s) {
    constexpr int G = 8;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(t, 8 * (32 / G)), 148 * 16));
    LOVE_LAUNCH((add_predict_kernel<V, G>), blocks, 256, 0, s, c.ad, (const double*)c.cols64, c.prior, (const V*)c.Rc,
                c.k_pad, (const double*)c.a, Xa, Xb, t, out, mean_out, c.counters);
}

template void add_scatter<float>(const Cache&, const float*, StepRef, double*, cudaStream_t);
template void add_scatter<double>(const Cache&, const double*, StepRef, double*, cudaStream_t);
template void add_gather<float>(const Cache&, const double*, const float*, StepRef, float*, double*, cudaStream_t,
                                const RcStream*);
template void add_gather<double>(const Cache&, const double*, const double*, StepRef, double*, double*, cudaStream_t,
                                 const RcStream*);
template void add_predict<float>(const Cache&, const double*, const double*, int64_t, float*, float*, cudaStream_t);
template void add_predict<double>(const Cache&, const double*, const double*, int64_t, double*, double*,
                                  cudaStream_t);

}  // namespace love
