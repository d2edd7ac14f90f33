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

#include "love_internal.h"

namespace love {

namespace {

template <int D> struct Slots { static constexpr int value = 1 << (2 * D); };

template <typename V, int D>
__global__ void __launch_bounds__(256) moments_kernel(int64_t n_items, const int* __restrict__ item_start,
                                                      const V* __restrict__ f0, const V* __restrict__ f1,
                                                      const V* __restrict__ f2, const V* __restrict__ q,
                                                      V* __restrict__ M) {
    constexpr int S = Slots<D>::value;
    const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (it >= n_items) return;
    const int p0 = item_start[it], p1 = item_start[it + 1];
    V acc[S];
#pragma unroll
    for (int l = 0; l < S; ++l) acc[l] = V(0);
    for (int p = p0; p < p1; ++p) {
        const V qv = q[p];
        V w0[4], w1[4], w2[4];
        keys4<V>(f0[p], w0);
        if (D > 1) keys4<V>(f1[p], w1);
        if (D > 2) keys4<V>(f2[p], w2);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const V ta = qv * w0[a];
            if (D == 1) {
                acc[a] += ta;
            } else {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const V tb = ta * w1[b];
                    if (D == 2) {
                        acc[a * 4 + b] += tb;
                    } else {
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) acc[(a * 4 + b) * 4 + cc] += tb * w2[cc];
                    }
                }
            }
        }
    }
#pragma unroll
    for (int l = 0; l < S; ++l) M[(int64_t)l * n_items + it] = acc[l];
}

// u[i] = scale * sum over slots l of sum over items of cell (i - l + 1) of M[l][item]
template <typename V, int D>
__global__ void __launch_bounds__(256) nodepass_kernel(GridDev g, int64_t n_items,
                                                       const int* __restrict__ cis,
                                                       const V* __restrict__ M,
                                                       const double* __restrict__ scale,
                                                       V* __restrict__ u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.m_total) return;
    int ic[3] = {0, 0, 0};
    {
        int rem = i;
        for (int d = 0; d < D; ++d) {
            ic[d] = rem / g.stride[d];
            rem -= ic[d] * g.stride[d];
        }
    }
    V sum = V(0);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int c0 = ic[0] - a + 1;
        if (c0 < 0 || c0 >= g.m[0]) continue;
        if (D == 1) {
            const int cf = c0;
            const int e = cis[cf + 1];
            for (int it = cis[cf]; it < e; ++it) sum += M[(int64_t)a * n_items + it];
            continue;
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int c1 = ic[1] - b + 1;
            if (c1 < 0 || c1 >= g.m[1]) continue;
            if (D == 2) {
                const int cf = c0 * g.stride[0] + c1;
                const int e = cis[cf + 1];
                for (int it = cis[cf]; it < e; ++it) sum += M[(int64_t)(a * 4 + b) * n_items + it];
                continue;
            }
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int c2 = ic[2] - cc + 1;
                if (c2 < 0 || c2 >= g.m[2]) continue;
                const int cf = c0 * g.stride[0] + c1 * g.stride[1] + c2;
                const int e = cis[cf + 1];
                for (int it = cis[cf]; it < e; ++it)
                    sum += M[(int64_t)((a * 4 + b) * 4 + cc) * n_items + it];
            }
        }
    }
    u[i] = (V)((double)sum * (*scale));
}

template <typename V, int D>
__global__ void __launch_bounds__(256) gather_kernel(GridDev g, int64_t n_items,
                                                     const int* __restrict__ item_cell,
                                                     const int* __restrict__ item_start,
                                                     const V* __restrict__ f0, const V* __restrict__ f1,
                                                     const V* __restrict__ f2, const V* __restrict__ z,
                                                     const V* __restrict__ q,
                                                     const double* __restrict__ qscale, double sigma2,
                                                     V* __restrict__ r, double* __restrict__ alpha_acc) {
    constexpr int S = Slots<D>::value;
    __shared__ double red[32];
    const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const double sc = *qscale;
    const V vsc = (V)sc, vsig = (V)(sigma2 * sc);
    double alpha = 0.0;
    if (it < n_items) {
        const int c = item_cell[it];
        int base = 0;
        {
            int rem = c;
            for (int d = 0; d < D; ++d) {
                const int cd = rem / g.stride[d];
                rem -= cd * g.stride[d];
                base += (cd - 1) * g.stride[d];
            }
        }
        V zl[S];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            if (D == 1) {
                zl[a] = z[base + a];
            } else {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if (D == 2) {
                        zl[a * 4 + b] = z[base + a * g.stride[0] + b];
                    } else {
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc)
                            zl[(a * 4 + b) * 4 + cc] = z[base + a * g.stride[0] + b * g.stride[1] + cc];
                    }
                }
            }
        }
        const int p0 = item_start[it], p1 = item_start[it + 1];
        for (int p = p0; p < p1; ++p) {
            V w0[4], w1[4], w2[4];
            keys4<V>(f0[p], w0);
            if (D > 1) keys4<V>(f1[p], w1);
            if (D > 2) keys4<V>(f2[p], w2);
            V acc = V(0);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                if (D == 1) {
                    acc += w0[a] * zl[a];
                } else {
                    V ta = V(0);
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        if (D == 2) {
                            ta += w1[b] * zl[a * 4 + b];
                        } else {
                            V tb = V(0);
#pragma unroll
                            for (int cc = 0; cc < 4; ++cc) tb += w2[cc] * zl[(a * 4 + b) * 4 + cc];
                            ta += w1[b] * tb;
                        }
                    }
                    acc += w0[a] * ta;
                }
            }
            const V qv = q[p];
            const V rv = acc + vsig * qv;
            r[p] = rv;
            alpha += (double)(vsc * qv) * (double)rv;
        }
    }
    if (alpha_acc != nullptr) {
        alpha = block_sum(alpha, red);
        if (threadIdx.x == 0) atomicAdd(alpha_acc, alpha);
    }
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

}  // namespace

template <typename V>
void launch_scatter(const Cache& c, const V* q, const double* scale, V* u, cudaStream_t s) {
    const int64_t ni = c.n_items;
    const int mt = c.g.m_total;
    const int gi = (int)std::max<int64_t>(1, ceil_div(ni, 256));
    const int gm = (int)ceil_div(mt, 256);
    const V* f0 = (const V*)c.frac[0];
    const V* f1 = (const V*)c.frac[1];
    const V* f2 = (const V*)c.frac[2];
    V* M = (V*)c.M;
    switch (c.g.d) {
        case 1:
            if (ni) LOVE_LAUNCH((moments_kernel<V, 1>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, M);
            LOVE_LAUNCH((nodepass_kernel<V, 1>), gm, 256, 0, s, c.g, ni, c.cell_item_start, M, scale, u);
            break;
        case 2:
            if (ni) LOVE_LAUNCH((moments_kernel<V, 2>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, M);
            LOVE_LAUNCH((nodepass_kernel<V, 2>), gm, 256, 0, s, c.g, ni, c.cell_item_start, M, scale, u);
            break;
        default:
            if (ni) LOVE_LAUNCH((moments_kernel<V, 3>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, M);
            LOVE_LAUNCH((nodepass_kernel<V, 3>), gm, 256, 0, s, c.g, ni, c.cell_item_start, M, scale, u);
            break;
    }
}

template <typename V>
void launch_gather(const Cache& c, const V* z, const V* q, const double* qscale, V* r,
                   double* alpha_acc, cudaStream_t s) {
    const int64_t ni = c.n_items;
    if (ni == 0) return;
    const int gi = (int)ceil_div(ni, 256);
    const V* f0 = (const V*)c.frac[0];
    const V* f1 = (const V*)c.frac[1];
    const V* f2 = (const V*)c.frac[2];
    switch (c.g.d) {
        case 1:
            LOVE_LAUNCH((gather_kernel<V, 1>), gi, 256, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1,
                        f2, z, q, qscale, c.sigma2, r, alpha_acc);
            break;
        case 2:
            LOVE_LAUNCH((gather_kernel<V, 2>), gi, 256, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1,
                        f2, z, q, qscale, c.sigma2, r, alpha_acc);
            break;
        default:
            LOVE_LAUNCH((gather_kernel<V, 3>), gi, 256, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1,
                        f2, z, q, qscale, c.sigma2, r, alpha_acc);
            break;
    }
}

template <typename V>
void launch_permute(const Cache& c, const V* in, V* out, bool to_sorted, cudaStream_t s) {
    if (c.n == 0) return;
    const int gb = (int)std::min<int64_t>(ceil_div(c.n, 256), 148 * 32);
    LOVE_LAUNCH(permute_kernel<V>, gb, 256, 0, s, c.perm, c.n, in, out, to_sorted ? 1 : 0);
}

template void launch_scatter<float>(const Cache&, const float*, const double*, float*, cudaStream_t);
template void launch_scatter<double>(const Cache&, const double*, const double*, double*, cudaStream_t);
template void launch_gather<float>(const Cache&, const float*, const float*, const double*, float*,
                                   double*, cudaStream_t);
template void launch_gather<double>(const Cache&, const double*, const double*, const double*, double*,
                                    double*, cudaStream_t);
template void launch_permute<float>(const Cache&, const float*, float*, bool, cudaStream_t);
template void launch_permute<double>(const Cache&, const double*, double*, bool, cudaStream_t);

}  // namespace love
