// ski_device.cuh -- device building blocks of the SKI interpolation operators,
// shared by the stand-alone scatter/gather kernels (ski.cu) and the fused Lanczos pass.
#pragma once
#include <type_traits>

#include "love_internal.h"

namespace love {

template <int D> struct Slots { static constexpr int value = 1 << (2 * D); };

// arithmetic type of per-point stencil sums: fp64 for d <= 2 (m-side precision plan), V for
// the 64-slot 3-D stencil (registers; 3-D configs are far from the cancellation regime)
template <typename V, int D> struct AccT { using type = double; };
template <int D> struct AccT<float, D> { using type = typename std::conditional<D == 3, float, double>::type; };

// flat index of the stencil origin (cell - 1 in every dimension) of flat cell c
template <int D>
__device__ __forceinline__ int stencil_base(const GridDev& g, int c) {
    int base = 0, rem = c;
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int cd = rem / g.stride[d];
        rem -= cd * g.stride[d];
        base += (cd - 1) * g.stride[d];
    }
    return base;
}

// the 4^d values of z on the stencil of a cell (slot order row-major, last dim fastest)
template <typename A, int D>
__device__ __forceinline__ void load_stencil(const GridDev& g, const double* __restrict__ z, int base,
                                             A zl[Slots<D>::value]) {
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
}

// w_x^T z_stencil with the tensor-product Keys weights
template <typename A, int D>
__device__ __forceinline__ A stencil_dot(const A w0[4], const A w1[4], const A w2[4], const A zl[Slots<D>::value]) {
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
    return acc;
}

// acc_l += v * w_l over the 4^d slots (stencil moments of one point)
template <typename A, int D>
__device__ __forceinline__ void stencil_accum(A acc[Slots<D>::value], A v, const A w0[4], const A w1[4],
                                              const A w2[4]) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const A ta = v * w0[a];
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

// ---- packed fp32 pairs (Blackwell FFMA2: fma.rn.f32x2).  A pair lives in one 64-bit
// register; a scalar operand packed as {x, x} is folded by ptxas into a broadcast operand.
// Per lane the result is the scalar FMA's, bit for bit.
using f32x2 = unsigned long long;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float lo2(f32x2 v) {
    float a;
    asm("{.reg .f32 t; mov.b64 {%0, t}, %1;}" : "=f"(a) : "l"(v));
    return a;
}
__device__ __forceinline__ float hi2(f32x2 v) {
    float b;
    asm("{.reg .f32 t; mov.b64 {t, %0}, %1;}" : "=f"(b) : "l"(v));
    return b;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// w^T z over the 64-node stencil for TWO points of the same cell (the 3-D fp32 gather):
// the same FMA sequence as stencil_dot<float, 3> per point, two points per instruction
__device__ __forceinline__ f32x2 stencil_dot3_pair(const f32x2 w0[4], const f32x2 w1[4], const f32x2 w2[4],
                                                   const float zl[64]) {
    f32x2 acc = 0ull;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        f32x2 ta = 0ull;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            f32x2 tb = 0ull;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const float zv = zl[(a * 4 + b) * 4 + cc];
                tb = fma2(w2[cc], pk2(zv, zv), tb);
            }
            ta = fma2(w1[b], tb, ta);
        }
        acc = fma2(w0[a], ta, acc);
    }
    return acc;
}

// (W v)[i] = sum over slots l of the moments M[l][item] of the items of cell i - l + 1
template <int D>
__device__ __forceinline__ double node_pull(const GridDev& g, int64_t n_items, const int* __restrict__ cis,
                                            const double* __restrict__ M, int i) {
    int ic[3] = {0, 0, 0};
    {
        int rem = i;
#pragma unroll
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
            const int e = cis[c0 + 1];
            for (int it = cis[c0]; it < e; ++it) sum += M[(int64_t)a * n_items + it];
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
                for (int it = cis[cf]; it < e; ++it) sum += M[(int64_t)((a * 4 + b) * 4 + cc) * n_items + it];
            }
        }
    }
    return sum;
}

}  // namespace love
