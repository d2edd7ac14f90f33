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

#include <type_traits>

#include "love_internal.h"

namespace love {

namespace {

template <int D> struct Slots { static constexpr int value = 1 << (2 * D); };

// arithmetic type of the per-point stencil sums: fp64 for d <= 2 (m-side precision plan),
// V for the 64-slot 3-D stencil (registers; 3-D configs are far from the cancellation regime)
template <typename V, int D> struct AccT { using type = double; };
template <int D> struct AccT<float, D> { using type = typename std::conditional<D == 3, float, double>::type; };

template <typename V, int D>
__global__ void __launch_bounds__(256) moments_kernel(int64_t n_items, const int* __restrict__ item_start,
                                                      const V* __restrict__ f0, const V* __restrict__ f1,
                                                      const V* __restrict__ f2, const V* __restrict__ qbase,
                                                      StepRef ref, double* __restrict__ M) {
    using A = typename AccT<V, D>::type;
    constexpr int S = Slots<D>::value;
    const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (it >= n_items || step_done(ref)) return;
    const V* __restrict__ q = qbase + step_j(ref) * ref.ld;
    const int p0 = item_start[it], p1 = item_start[it + 1];
    A acc[S];
#pragma unroll
    for (int l = 0; l < S; ++l) acc[l] = A(0);
    constexpr int B = 8;                    // points loaded per batch (memory-level parallelism)
    for (int pb = p0; pb < p1; pb += B) {
        A qv[B], fa[B], fb[B], fc[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int p = pb + u;
            const bool in = p < p1;
            qv[u] = in ? (A)q[p] : A(0);    // q = 0 makes padded lanes contribute nothing
            fa[u] = in ? (A)f0[p] : A(0);
            fb[u] = (D > 1 && in) ? (A)f1[p] : A(0);
            fc[u] = (D > 2 && in) ? (A)f2[p] : A(0);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            A w0[4], w1[4], w2[4];
            keys4<A>(fa[u], w0);
            if (D > 1) keys4<A>(fb[u], w1);
            if (D > 2) keys4<A>(fc[u], w2);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const A ta = qv[u] * w0[a];
                if (D == 1) {
                    acc[a] += ta;
                } else {
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const A tb = ta * w1[b];
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
    }
#pragma unroll
    for (int l = 0; l < S; ++l) M[(int64_t)l * n_items + it] = (double)acc[l];
}

// u[i] = scale * sum over slots l of sum over items of cell (i - l + 1) of M[l][item]
template <int D>
__global__ void __launch_bounds__(256) nodepass_kernel(GridDev g, int64_t n_items,
                                                       const int* __restrict__ cis,
                                                       const double* __restrict__ M, StepRef ref,
                                                       double* __restrict__ u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.m_total || step_done(ref)) return;
    int ic[3] = {0, 0, 0};
    {
        int rem = i;
        for (int d = 0; d < D; ++d) {
            ic[d] = rem / g.stride[d];
            rem -= ic[d] * g.stride[d];
        }
    }
    double sum = 0.0;
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
    u[i] = sum * ref.scale[step_j(ref)];
}

template <typename V, int D>
__global__ void __launch_bounds__(256) gather_kernel(GridDev g, int64_t n_items,
                                                     const int* __restrict__ item_cell,
                                                     const int* __restrict__ item_start,
                                                     const V* __restrict__ f0, const V* __restrict__ f1,
                                                     const V* __restrict__ f2, const double* __restrict__ z,
                                                     const V* __restrict__ qbase, StepRef ref, double sigma2,
                                                     V* __restrict__ r, double* __restrict__ alpha_base) {
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
        A zl[S];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            if (D == 1) {
                zl[a] = (A)z[base + a];
            } else {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if (D == 2) {
                        zl[a * 4 + b] = (A)z[base + a * g.stride[0] + b];
                    } else {
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc)
                            zl[(a * 4 + b) * 4 + cc] = (A)z[base + a * g.stride[0] + b * g.stride[1] + cc];
                    }
                }
            }
        }
        const int p0 = item_start[it], p1 = item_start[it + 1];
        constexpr int B = 8;                // points loaded per batch
        for (int pb = p0; pb < p1; pb += B) {
            A qv[B], fa[B], fb[B], fc[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int p = pb + u;
                const bool in = p < p1;
                qv[u] = in ? (A)q[p] : A(0);
                fa[u] = in ? (A)f0[p] : A(0);
                fb[u] = (D > 1 && in) ? (A)f1[p] : A(0);
                fc[u] = (D > 2 && in) ? (A)f2[p] : A(0);
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                A w0[4], w1[4], w2[4];
                keys4<A>(fa[u], w0);
                if (D > 1) keys4<A>(fb[u], w1);
                if (D > 2) keys4<A>(fc[u], w2);
                A acc = A(0);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    if (D == 1) {
                        acc += w0[a] * zl[a];
                    } else {
                        A ta = A(0);
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            if (D == 2) {
                                ta += w1[b] * zl[a * 4 + b];
                            } else {
                                A tb = A(0);
#pragma unroll
                                for (int cc = 0; cc < 4; ++cc) tb += w2[cc] * zl[(a * 4 + b) * 4 + cc];
                                ta += w1[b] * tb;
                            }
                        }
                        acc += w0[a] * ta;
                    }
                }
                const V rv = (V)(acc + vsig * qv[u]);
                if (pb + u < p1) {
                    r[pb + u] = rv;
                    alpha += (double)(vsc * qv[u]) * (double)rv;
                }
            }
        }
    }
    if (alpha_base != nullptr) {
        alpha = block_sum(alpha, red);
        if (threadIdx.x == 0) atomicAdd(alpha_base + j, alpha);
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
void launch_scatter(const Cache& c, const V* q, StepRef ref, double* u, cudaStream_t s) {
    const int64_t ni = c.n_items;
    const int mt = c.g.m_total;
    const int gi = (int)std::max<int64_t>(1, ceil_div(ni, 256));
    const int gm = (int)ceil_div(mt, 256);
    const V* f0 = (const V*)c.frac[0];
    const V* f1 = (const V*)c.frac[1];
    const V* f2 = (const V*)c.frac[2];
    double* M = (double*)c.M;
    switch (c.g.d) {
        case 1:
            if (ni) LOVE_LAUNCH((moments_kernel<V, 1>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, ref, M);
            LOVE_LAUNCH((nodepass_kernel<1>), gm, 256, 0, s, c.g, ni, c.cell_item_start, M, ref, u);
            break;
        case 2:
            if (ni) LOVE_LAUNCH((moments_kernel<V, 2>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, ref, M);
            LOVE_LAUNCH((nodepass_kernel<2>), gm, 256, 0, s, c.g, ni, c.cell_item_start, M, ref, u);
            break;
        default:
            if (ni) LOVE_LAUNCH((moments_kernel<V, 3>), gi, 256, 0, s, ni, c.item_start, f0, f1, f2, q, ref, M);
            LOVE_LAUNCH((nodepass_kernel<3>), gm, 256, 0, s, c.g, ni, c.cell_item_start, M, ref, u);
            break;
    }
}

template <typename V>
void launch_gather(const Cache& c, const double* z, const V* q, StepRef ref, V* r, double* alpha_base,
                   cudaStream_t s) {
    const int64_t ni = c.n_items;
    if (ni == 0) return;
    const int gi = (int)ceil_div(ni, 256);
    const V* f0 = (const V*)c.frac[0];
    const V* f1 = (const V*)c.frac[1];
    const V* f2 = (const V*)c.frac[2];
    switch (c.g.d) {
        case 1:
            LOVE_LAUNCH((gather_kernel<V, 1>), gi, 256, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1,
                        f2, z, q, ref, c.sigma2, r, alpha_base);
            break;
        case 2:
            LOVE_LAUNCH((gather_kernel<V, 2>), gi, 256, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1,
                        f2, z, q, ref, c.sigma2, r, alpha_base);
            break;
        default:
            LOVE_LAUNCH((gather_kernel<V, 3>), gi, 256, 0, s, c.g, ni, c.item_cell, c.item_start, f0, f1,
                        f2, z, q, ref, c.sigma2, r, alpha_base);
            break;
    }
}

template <typename V>
void launch_permute(const Cache& c, const V* in, V* out, bool to_sorted, cudaStream_t s) {
    if (c.n == 0) return;
    const int gb = (int)std::min<int64_t>(ceil_div(c.n, 256), 148 * 32);
    LOVE_LAUNCH(permute_kernel<V>, gb, 256, 0, s, c.perm, c.n, in, out, to_sorted ? 1 : 0);
}

template <typename A, typename B>
__global__ void convert_kernel(const A* __restrict__ in, B* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (B)in[i];
}

template <typename A, typename B>
void launch_convert(const A* in, B* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    LOVE_LAUNCH((convert_kernel<A, B>), (int)std::min<int64_t>(ceil_div(n, 256), 148 * 16), 256, 0, s, in, out, n);
}

template void launch_convert<float, double>(const float*, double*, int64_t, cudaStream_t);
template void launch_convert<double, float>(const double*, float*, int64_t, cudaStream_t);
template void launch_scatter<float>(const Cache&, const float*, StepRef, double*, cudaStream_t);
template void launch_scatter<double>(const Cache&, const double*, StepRef, double*, cudaStream_t);
template void launch_gather<float>(const Cache&, const double*, const float*, StepRef, float*, double*,
                                   cudaStream_t);
template void launch_gather<double>(const Cache&, const double*, const double*, StepRef, double*, double*,
                                    cudaStream_t);
template void launch_permute<float>(const Cache&, const float*, float*, bool, cudaStream_t);
template void launch_permute<double>(const Cache&, const double*, double*, bool, cudaStream_t);

}  // namespace love
