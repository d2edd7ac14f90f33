// kuu.cu -- structured K_UU MVMs on the regular grid.
//
// d = 1 (Toeplitz): K_UU u = first m entries of IFFT(lambda * FFT([u; 0])) with the circulant
//   embedding of length N = 2^ceil(log2(2m-1)) (reading A25).  Hand-written shared-memory
//   radix-2 Stockham FFTs: one CTA for N <= 4096 (fp32) / 2048 (fp64), otherwise the
//   four-step factorisation N = N1 * N2 in three passes whose middle pass does
//   forward FFT -> multiply by lambda -> inverse FFT on the same smem lines (no transposes).
//   lambda (scaled by s^2/N) is computed once per build with the same kernels in fp64.
// d > 1 (Kronecker of Toeplitz): T(c_d) applied along each axis by a dense per-axis
//   product from shared memory (m_d <= 1024: m * m_d FMAs per axis, exact, no FFT round-off).
#include <cuda_runtime.h>

#include <cmath>

#include "love_internal.h"

namespace love {

namespace {

template <typename R> struct Cx;
template <> struct Cx<float> { using T = float2; };
template <> struct Cx<double> { using T = double2; };

template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
    C r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}

__device__ __forceinline__ void sincospi_t(float x, float* s, float* c) { sincospif(x, s, c); }
__device__ __forceinline__ void sincospi_t(double x, double* s, double* c) { sincospi(x, s, c); }

// exp(sign * 2 pi i * num / den) for integers 0 <= num < den (den a power of two), exact
// argument reduction in integer arithmetic.
template <typename R>
__device__ __forceinline__ typename Cx<R>::T twiddle(int64_t num, int64_t den, int sign) {
    typename Cx<R>::T w;
    R s, c;
    sincospi_t((R)(2.0 * (double)num / (double)den), &s, &c);
    w.x = c;
    w.y = sign < 0 ? -s : s;
    return w;
}

// Radix-2 Stockham autosort FFT of G lines of length L (= 1 << logL) stored contiguously in
// `a` (line g at a + g*L), `b` same-size scratch, tw[k] = exp(-2 pi i k / L), k < L/2.
// sign = -1 forward, +1 inverse (unnormalised).  Returns the buffer holding the result.
template <typename C>
__device__ C* stockham(C* a, C* b, const C* tw, int G, int L, int logL, int sign) {
    const int half = L >> 1;
    for (int Ns = 1, s = 0; Ns < L; Ns <<= 1, ++s) {
        const int tstep = L / (2 * Ns);   // twiddle table stride for this stage
        for (int t = threadIdx.x; t < G * half; t += blockDim.x) {
            const int line = t >> (logL - 1);
            const int j = t & (half - 1);
            const C* src = a + line * L;
            C* dst = b + line * L;
            const int k = j & (Ns - 1);
            const C v0 = src[j];
            C w = tw[k * tstep];
            if (sign > 0) w.y = -w.y;
            const C v1 = cmul(src[j + half], w);
            const int idxD = ((j - k) << 1) + k;
            C o0, o1;
            o0.x = v0.x + v1.x; o0.y = v0.y + v1.y;
            o1.x = v0.x - v1.x; o1.y = v0.y - v1.y;
            dst[idxD] = o0;
            dst[idxD + Ns] = o1;
        }
        __syncthreads();
        C* tmp = a; a = b; b = tmp;
    }
    return a;
}

template <typename R>
__device__ void fill_twiddles(typename Cx<R>::T* tw, int L) {
    for (int k = threadIdx.x; k < L / 2; k += blockDim.x) tw[k] = twiddle<R>(k, L, -1);
}

// ---- single-CTA convolution / forward transform (N small)
// mode 0: z[n] = Re IFFT(lam * FFT([u;0]))[n], n < m   (lam already holds s^2/N)
// mode 1: outc[k] = FFT(u)[k] (u has N entries)                      (lambda setup)
template <typename R>
__global__ void fft_small_kernel(const R* __restrict__ u, int m, int N, int logN,
                                 const R* __restrict__ lam, R* __restrict__ z,
                                 typename Cx<R>::T* __restrict__ outc, int mode) {
    using C = typename Cx<R>::T;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* a = (C*)smraw;
    C* b = a + N;
    C* tw = b + N;
    fill_twiddles<R>(tw, N);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        C v;
        v.x = i < m ? u[i] : R(0);
        v.y = R(0);
        a[i] = v;
    }
    __syncthreads();
    C* x = stockham<C>(a, b, tw, 1, N, logN, -1);
    if (mode == 1) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) outc[i] = x[i];
        return;
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const R l = lam[i];
        x[i].x *= l;
        x[i].y *= l;
    }
    __syncthreads();
    C* y = stockham<C>(x, x == a ? b : a, tw, 1, N, logN, +1);
    for (int i = threadIdx.x; i < m; i += blockDim.x) z[i] = y[i].x;
}

// ---- four-step pass A: for each n1, FFT over n2 of x[n1 + N1 n2], times w_N^{n1 k2}
template <typename R, int G>
__global__ void fft_passA_kernel(const R* __restrict__ u, int m, int N1, int N2, int logN2,
                                 typename Cx<R>::T* __restrict__ Y) {
    using C = typename Cx<R>::T;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* a = (C*)smraw;
    C* b = a + G * N2;
    C* tw = b + G * N2;
    fill_twiddles<R>(tw, N2);
    const int n1_0 = blockIdx.x * G;
    const int64_t N = (int64_t)N1 * N2;
    for (int t = threadIdx.x; t < G * N2; t += blockDim.x) {
        const int g = t % G, n2 = t / G;
        const int64_t idx = n1_0 + g + (int64_t)N1 * n2;
        C v;
        v.x = idx < m ? u[idx] : R(0);
        v.y = R(0);
        a[g * N2 + n2] = v;
    }
    __syncthreads();
    C* x = stockham<C>(a, b, tw, G, N2, logN2, -1);
    for (int t = threadIdx.x; t < G * N2; t += blockDim.x) {
        const int g = t / N2, k2 = t % N2;
        const int n1 = n1_0 + g;
        const C w = twiddle<R>(((int64_t)n1 * k2) % N, N, -1);
        Y[(int64_t)n1 * N2 + k2] = cmul(x[g * N2 + k2], w);
    }
}

// ---- four-step pass B: for each k2, FFT over n1 -> X[N2 k1 + k2];
// mode 0: multiply by lamB[k2*N1 + k1], inverse FFT over k1, times w_N^{-n1 k2}, store back
// mode 1: store X in natural order into outc
template <typename R, int G>
__global__ void fft_passB_kernel(typename Cx<R>::T* __restrict__ Y, int N1, int N2, int logN1,
                                 const R* __restrict__ lamB, typename Cx<R>::T* __restrict__ outc,
                                 int mode) {
    using C = typename Cx<R>::T;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* a = (C*)smraw;
    C* b = a + G * N1;
    C* tw = b + G * N1;
    fill_twiddles<R>(tw, N1);
    const int k2_0 = blockIdx.x * G;
    const int64_t N = (int64_t)N1 * N2;
    for (int t = threadIdx.x; t < G * N1; t += blockDim.x) {
        const int g = t % G, n1 = t / G;
        a[g * N1 + n1] = Y[(int64_t)n1 * N2 + k2_0 + g];
    }
    __syncthreads();
    C* x = stockham<C>(a, b, tw, G, N1, logN1, -1);
    if (mode == 1) {
        for (int t = threadIdx.x; t < G * N1; t += blockDim.x) {
            const int g = t % G, k1 = t / G;
            outc[(int64_t)N2 * k1 + k2_0 + g] = x[g * N1 + k1];
        }
        return;
    }
    for (int t = threadIdx.x; t < G * N1; t += blockDim.x) {
        const int g = t / N1, k1 = t % N1;
        const R l = lamB[(int64_t)(k2_0 + g) * N1 + k1];
        x[t].x *= l;
        x[t].y *= l;
    }
    __syncthreads();
    C* y = stockham<C>(x, x == a ? b : a, tw, G, N1, logN1, +1);
    for (int t = threadIdx.x; t < G * N1; t += blockDim.x) {
        const int g = t % G, n1 = t / G;
        const int k2 = k2_0 + g;
        const C w = twiddle<R>(((int64_t)n1 * k2) % N, N, +1);
        Y[(int64_t)n1 * N2 + k2] = cmul(y[g * N1 + n1], w);
    }
}

// ---- four-step pass A': for each n1, inverse FFT over k2; z[n1 + N1 n2] = Re(.)
template <typename R, int G>
__global__ void fft_passC_kernel(const typename Cx<R>::T* __restrict__ Y, int m, int N1, int N2,
                                 int logN2, R* __restrict__ z) {
    using C = typename Cx<R>::T;
    extern __shared__ __align__(16) unsigned char smraw[];
    C* a = (C*)smraw;
    C* b = a + G * N2;
    C* tw = b + G * N2;
    fill_twiddles<R>(tw, N2);
    const int n1_0 = blockIdx.x * G;
    for (int t = threadIdx.x; t < G * N2; t += blockDim.x) {
        const int g = t / N2, k2 = t % N2;
        a[t] = Y[(int64_t)(n1_0 + g) * N2 + k2];
    }
    __syncthreads();
    C* x = stockham<C>(a, b, tw, G, N2, logN2, +1);
    for (int t = threadIdx.x; t < G * N2; t += blockDim.x) {
        const int g = t % G, n2 = t / G;
        const int64_t idx = n1_0 + g + (int64_t)N1 * n2;
        if (idx < m) z[idx] = x[g * N2 + n2].x;
    }
}

// ---- dense per-axis Toeplitz products (d > 1)
// layout (outer O, length L, inner I): out(o,l,i) = scale * sum_l' c[|l-l'|] in(o,l',i)
template <typename V>
__global__ void axis_inner_kernel(const V* __restrict__ in, V* __restrict__ out,
                                  const V* __restrict__ c, int L, int I, int RL, V scale) {
    extern __shared__ __align__(16) unsigned char smraw[];
    V* cs = (V*)smraw;           // [L]
    V* tile = cs + L;            // [L][32]
    const int i0 = blockIdx.x * 32;
    const int r0 = blockIdx.y * RL;
    const int64_t ob = (int64_t)blockIdx.z * L * I;
    for (int t = threadIdx.x; t < L; t += blockDim.x) cs[t] = c[t];
    for (int t = threadIdx.x; t < L * 32; t += blockDim.x) {
        const int l = t >> 5, ii = t & 31;
        tile[t] = (i0 + ii < I) ? in[ob + (int64_t)l * I + i0 + ii] : V(0);
    }
    __syncthreads();
    const int ii = threadIdx.x & 31;
    for (int r = r0 + (threadIdx.x >> 5); r < min(L, r0 + RL); r += blockDim.x >> 5) {
        V acc = V(0);
        for (int l = 0; l < L; ++l) acc += cs[abs(r - l)] * tile[l * 32 + ii];
        if (i0 + ii < I) out[ob + (int64_t)r * I + i0 + ii] = acc * scale;
    }
}

template <typename V>
__global__ void axis_line_kernel(const V* __restrict__ in, V* __restrict__ out,
                                 const V* __restrict__ c, int O, int L, int LPB, V scale) {
    extern __shared__ __align__(16) unsigned char smraw[];
    V* cs = (V*)smraw;           // [L]
    V* lines = cs + L;           // [LPB][L]
    const int64_t o0 = (int64_t)blockIdx.x * LPB;
    const int nl = (int)(((int64_t)LPB < (int64_t)O - o0) ? (int64_t)LPB : (int64_t)O - o0);
    for (int t = threadIdx.x; t < L; t += blockDim.x) cs[t] = c[t];
    for (int t = threadIdx.x; t < nl * L; t += blockDim.x) lines[t] = in[o0 * L + t];
    __syncthreads();
    for (int t = threadIdx.x; t < nl * L; t += blockDim.x) {
        const int ln = t / L, r = t % L;
        const V* x = lines + ln * L;
        V acc = V(0);
        for (int l = 0; l < L; ++l) acc += cs[abs(r - l)] * x[l];
        out[o0 * L + t] = acc * scale;
    }
}

__global__ void rbf_columns_kernel(GridDev g, double l0, double l1, double l2, double* __restrict__ cols) {
    const double ls[3] = {l0, l1, l2};
    int off = 0;
    for (int d = 0; d < g.d; ++d) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.m[d]; i += gridDim.x * blockDim.x) {
            const double r = (double)i * g.h[d];
            cols[off + i] = exp(-(r * r) / (2.0 * ls[d] * ls[d]));   // c_d[i] (A6)
        }
        off += g.m[d];
    }
}

__global__ void embed_kernel(const double* __restrict__ c, int m, int N, double* __restrict__ col) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (i < m) v = c[i];
        else if (i > N - m) v = c[N - i];
        col[i] = v;
    }
}

template <typename V>
__global__ void lambda_store_kernel(const double2* __restrict__ X, int N, int N1, int N2, int four_step,
                                    double scale, V* __restrict__ lam) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const double v = X[k].x * scale;
        if (four_step) {
            const int k1 = k / N2, k2 = k % N2;   // k = N2 k1 + k2
            lam[(int64_t)k2 * N1 + k1] = (V)v;
        } else {
            lam[k] = (V)v;
        }
    }
}

template <typename V>
__global__ void cast_kernel(const double* __restrict__ a, V* __restrict__ b, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = (V)a[i];
}

inline int ilog2(int64_t x) {
    int l = 0;
    while ((int64_t(1) << l) < x) ++l;
    return l;
}

template <typename R> constexpr int lines_per_cta() { return sizeof(R) == 4 ? 4 : 2; }
template <typename R> int small_fft_max() { return sizeof(R) == 4 ? 4096 : 2048; }

template <typename R>
size_t fft_line_smem(int G, int L) {
    return sizeof(typename Cx<R>::T) * (size_t)(2 * G * L + L / 2);
}

template <typename R>
void set_smem_attr(const void* fn, size_t bytes) {
    if (bytes > 48 * 1024) cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)bytes), "smem attr");
}

// convolution (mode 0) of u (m entries) or forward FFT (mode 1) of u (N entries)
template <typename R>
void fft_run(int N, int N1, int N2, const R* u, int m, const R* lam, R* z,
             typename Cx<R>::T* work, typename Cx<R>::T* outc, int mode, cudaStream_t s) {
    using C = typename Cx<R>::T;
    if (N1 == 0) {
        const size_t sm = fft_line_smem<R>(1, N);
        set_smem_attr<R>((const void*)fft_small_kernel<R>, sm);
        LOVE_LAUNCH(fft_small_kernel<R>, 1, 1024, sm, s, u, m, N, ilog2(N), lam, z, outc, mode);
        return;
    }
    constexpr int G = lines_per_cta<R>();
    const size_t smA = fft_line_smem<R>(G, N2), smB = fft_line_smem<R>(G, N1);
    set_smem_attr<R>((const void*)fft_passA_kernel<R, G>, smA);
    set_smem_attr<R>((const void*)fft_passB_kernel<R, G>, smB);
    set_smem_attr<R>((const void*)fft_passC_kernel<R, G>, smA);
    LOVE_LAUNCH((fft_passA_kernel<R, G>), N1 / G, 256, smA, s, u, m, N1, N2, ilog2(N2), work);
    LOVE_LAUNCH((fft_passB_kernel<R, G>), N2 / G, 256, smB, s, work, N1, N2, ilog2(N1), lam, outc, mode);
    if (mode == 0)
        LOVE_LAUNCH((fft_passC_kernel<R, G>), N1 / G, 256, smA, s, (const C*)work, m, N1, N2, ilog2(N2), z);
}

template <typename V>
void kuu_axes(const Cache& c, const V* u, V* z, cudaStream_t s) {
    const GridDev& g = c.g;
    const V* in = u;
    int off = 0;
    for (int d = 0; d < g.d; ++d) {
        const int L = g.m[d];
        int O = 1, I = 1;
        for (int e = 0; e < d; ++e) O *= g.m[e];
        for (int e = d + 1; e < g.d; ++e) I *= g.m[e];
        V* out = (d == g.d - 1) ? z : (V*)c.ktmp[d & 1];
        const V scale = (d == g.d - 1) ? (V)c.rbf.outputscale : V(1);
        const V* col = (const V*)c.cols + off;
        if (I == 1) {
            const int LPB = std::max(1, 2048 / L);
            const size_t sm = sizeof(V) * (size_t)(L + LPB * L);
            set_smem_attr<V>((const void*)axis_line_kernel<V>, sm);
            LOVE_LAUNCH(axis_line_kernel<V>, (int)ceil_div(O, LPB), 256, sm, s, in, out, col, O, L, LPB, scale);
        } else {
            const int tiles = (int)ceil_div(I, 32);
            int RL = L;
            while (RL > 8 && (int64_t)tiles * O * ceil_div(L, RL) < 2 * 148) RL /= 2;
            const size_t sm = sizeof(V) * (size_t)(L + L * 32);
            set_smem_attr<V>((const void*)axis_inner_kernel<V>, sm);
            dim3 grid(tiles, (unsigned)ceil_div(L, RL), O);
            LOVE_LAUNCH(axis_inner_kernel<V>, grid, 256, sm, s, in, out, col, L, I, RL, scale);
        }
        in = out;
        off += L;
    }
}

}  // namespace

void setup_kuu(Cache& c, cudaStream_t s) {
    const GridDev& g = c.g;
    int msum = 0;
    for (int d = 0; d < g.d; ++d) msum += g.m[d];
    c.cols64 = (double*)dalloc(c, sizeof(double) * msum, s);
    c.cols = dalloc(c, c.vsize * msum, s);
    LOVE_LAUNCH(rbf_columns_kernel, 64, 256, 0, s, g, c.rbf.lengthscale[0], c.rbf.lengthscale[1],
                c.rbf.lengthscale[2], c.cols64);
    if (c.precision == LOVE_FP64) LOVE_LAUNCH(cast_kernel<double>, 64, 256, 0, s, c.cols64, (double*)c.cols, msum);
    else LOVE_LAUNCH(cast_kernel<float>, 64, 256, 0, s, c.cols64, (float*)c.cols, msum);

    if (g.d > 1) {
        for (int d = 0; d < g.d; ++d)
            if (g.m[d] > 1024) throw LoveError{LOVE_ERR_ARG, "Kronecker grids need m_d <= 1024 per axis"};
        c.ktmp[0] = dalloc(c, c.vsize * g.m_total, s);
        c.ktmp[1] = dalloc(c, c.vsize * g.m_total, s);
        return;
    }
    // d = 1: circulant embedding and its eigenvalues (fp64), stored * s^2 / N
    const int m = g.m[0];
    int N = 1;
    while (N < 2 * m - 1) N *= 2;
    if (N > (1 << 22)) throw LoveError{LOVE_ERR_ARG, "1-D grid too long (m <= 2^21)"};
    c.fft_N = N;
    const int small = (c.precision == LOVE_FP64) ? small_fft_max<double>() : small_fft_max<float>();
    if (N <= small) {
        c.fft_N1 = c.fft_N2 = 0;
    } else {
        const int lg = ilog2(N);
        c.fft_N1 = 1 << (lg / 2);
        c.fft_N2 = N / c.fft_N1;
    }
    c.lam = dalloc(c, c.vsize * N, s);
    c.fft_buf = dalloc(c, 2 * c.vsize * N, s);
    double* col = nullptr;
    double2* X = nullptr;
    double2* work = nullptr;
    cuda_check(cudaMallocAsync((void**)&col, sizeof(double) * N, s), "lam alloc");
    cuda_check(cudaMallocAsync((void**)&X, sizeof(double2) * N, s), "lam alloc");
    cuda_check(cudaMallocAsync((void**)&work, sizeof(double2) * N, s), "lam alloc");
    LOVE_LAUNCH(embed_kernel, (int)std::min<int64_t>(ceil_div(N, 256), 4096), 256, 0, s, c.cols64, m, N, col);
    // fp64 N1 may differ from the fp32 split only through the small-FFT threshold
    int N1 = c.fft_N1, N2 = c.fft_N2;
    if (N1 == 0 && N > small_fft_max<double>()) {
        const int lg = ilog2(N);
        N1 = 1 << (lg / 2);
        N2 = N / N1;
    }
    fft_run<double>(N, N1, N2, col, N, nullptr, nullptr, work, X, 1, s);
    const double scale = c.rbf.outputscale / (double)N;
    // the stored layout follows the split used by the vector-precision kernels
    const int four = c.fft_N1 != 0;
    if (c.precision == LOVE_FP64)
        LOVE_LAUNCH(lambda_store_kernel<double>, (int)std::min<int64_t>(ceil_div(N, 256), 4096), 256, 0, s, X, N,
                    c.fft_N1, c.fft_N2, four, scale, (double*)c.lam);
    else
        LOVE_LAUNCH(lambda_store_kernel<float>, (int)std::min<int64_t>(ceil_div(N, 256), 4096), 256, 0, s, X, N,
                    c.fft_N1, c.fft_N2, four, scale, (float*)c.lam);
    cuda_check(cudaFreeAsync(col, s), "lam free");
    cuda_check(cudaFreeAsync(X, s), "lam free");
    cuda_check(cudaFreeAsync(work, s), "lam free");
}

template <typename V>
void launch_kuu(const Cache& c, const V* u, V* z, cudaStream_t s) {
    if (c.g.d > 1) {
        kuu_axes<V>(c, u, z, s);
        return;
    }
    using C = typename Cx<V>::T;
    fft_run<V>(c.fft_N, c.fft_N1, c.fft_N2, u, c.g.m[0], (const V*)c.lam, z, (C*)c.fft_buf, nullptr, 0, s);
}

template void launch_kuu<float>(const Cache&, const float*, float*, cudaStream_t);
template void launch_kuu<double>(const Cache&, const double*, double*, cudaStream_t);

}  // namespace love
