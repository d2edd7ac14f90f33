// kuu.cu -- structured K_UU MVMs on the regular grid, fp64 on the m side.
//
// The m-sized side of the SKI MVM (u = W q, z = K_UU u) is always computed and stored in
// fp64, also in LOVE_FP32 mode: it is cheap (m << n) and it is what keeps fp32-mode
// variances inside the parity bound when var << prior ("Precision plan").
//
// d = 1 (Toeplitz): z = first m entries of IFFT(lambda * FFT([u; 0])) with the circulant
//   embedding of length N = 2^ceil(log2(2m-1)) (reading A25).  Hand-written shared-memory
//   Stockham FFTs with radix-8 register butterflies: one CTA for N <= 4096, otherwise the
//   four-step factorisation N = N1 * N2 in three passes whose middle pass does
//   forward FFT -> multiply by lambda -> inverse FFT on the same lines (no transposes).
//   lambda (times s^2 / N) is computed once per build with the same kernels.
// d > 1 (Kronecker of Toeplitz): T(c_d) applied along each axis by a dense per-axis
//   product from shared memory (m_d <= 1024: m * m_d FMAs per axis, no FFT round-off).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "love_internal.h"

namespace love {

LOVE_TRACE_TU(kuu)

namespace {

using C = double2;

__device__ __forceinline__ C cmul(C a, C b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ C cadd(C a, C b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ C csub(C a, C b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ C cconj(C a) { return make_double2(a.x, -a.y); }
// multiply by -i (SIGN < 0) or +i (SIGN > 0)
template <int SIGN> __device__ __forceinline__ C mul_i(C a) {
    return SIGN < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <int SIGN> __device__ __forceinline__ void dft2(C* v) {
    const C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <int SIGN> __device__ __forceinline__ void dft4(C& v0, C& v1, C& v2, C& v3) {
    const C t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = mul_i<SIGN>(csub(v1, v3));
    v0 = cadd(t0, t2);
    v1 = cadd(t1, t3);
    v2 = csub(t0, t2);
    v3 = csub(t1, t3);
}

template <int SIGN> __device__ __forceinline__ void dft8(C* v) {
    C e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    C o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<SIGN>(e0, e1, e2, e3);
    dft4<SIGN>(o0, o1, o2, o3);
    const double r = 0.70710678118654752440;
    // w^k = exp(SIGN * 2 pi i k / 8)
    const C w1 = make_double2(r, SIGN * r), w3 = make_double2(-r, SIGN * r);
    o1 = cmul(o1, w1);
    o2 = mul_i<SIGN>(o2);
    o3 = cmul(o3, w3);
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1); v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2); v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3); v[7] = csub(e3, o3);
}

// Shared-memory index with one double2 of padding every 8: the radix-8 Stockham stores of the
// first stage hit addresses 8 double2 (128 B) apart, which would all map to one bank group.
__device__ __forceinline__ int pad(int i) { return i + (i >> 3); }
inline size_t padded(size_t n) { return n + n / 8 + 1; }

// One radix-R stage of an in-place Stockham FFT over G lines of length L in shared memory
// (padded indices), run by a block of exactly G*L/EPT threads (EPT/R butterflies per thread).
// Every index into the register array is a compile-time constant (no local memory).
template <int SIGN, int R, int EPT = 8>
__device__ __forceinline__ void fft_stage(C* buf, int L, int Ns, const C* tw) {
    constexpr int PER = EPT / R;
    const int nb = L / R;                        // butterflies per line
    const int step = L / (Ns * R);               // twiddle stride
    C v[PER][R];
    int dst[PER];
#pragma unroll
    for (int c = 0; c < PER; ++c) {
        const int b = threadIdx.x + c * blockDim.x;
        const int line = b / nb, j = b - line * nb;
        const int k = j & (Ns - 1);
        const int base = line * L;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            C x = buf[pad(base + j + r * nb)];
            if (r > 0) {
                C w = tw[r * k * step];
                if (SIGN > 0) w = cconj(w);
                x = cmul(x, w);
            }
            v[c][r] = x;
        }
        dst[c] = base + (j - k) * R + k;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < PER; ++c) {
        if (R == 8) dft8<SIGN>(v[c]);
        else if (R == 4) dft4<SIGN>(v[c][0], v[c][1], v[c][2], v[c][3]);
        else dft2<SIGN>(v[c]);
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pad(dst[c] + r * Ns)] = v[c][r];
    }
    __syncthreads();
}

// In-place Stockham FFT of G lines of length L (contiguous in shared memory), run by a block
// of exactly G*L/8 threads: radix-8 stages while 8 divides the remaining length, then one
// radix-4 or radix-2 stage.  tw[k] = exp(-2 pi i k / L), k < L, in shared memory.
// SIGN = -1 forward, +1 inverse (unnormalised).
template <int SIGN>
__device__ void line_fft(C* buf, int L, const C* tw) {
    int Ns = 1;
    for (; Ns * 8 <= L; Ns *= 8) fft_stage<SIGN, 8>(buf, L, Ns, tw);
    if (Ns * 4 == L) fft_stage<SIGN, 4>(buf, L, Ns, tw);
    else if (Ns * 2 == L) fft_stage<SIGN, 2>(buf, L, Ns, tw);
}

// The same transform with 4 elements per thread (G*L/4 threads): radix-4 stages, then one
// radix-2 stage.  Twice the threads and a shorter dependent chain per thread than the radix-8
// form -- the axis passes run one 4-warp CTA per SM, where every fp64 latency is exposed.
template <int SIGN>
__device__ void line_fft4(C* buf, int L, const C* tw) {
    int Ns = 1;
    for (; Ns * 4 <= L; Ns *= 4) fft_stage<SIGN, 4, 4>(buf, L, Ns, tw);
    if (Ns * 2 == L) fft_stage<SIGN, 2, 4>(buf, L, Ns, tw);
}

// copy a line-length twiddle table from global to shared memory
__device__ __forceinline__ void load_tw(C* dst, const C* __restrict__ src, int L) {
    #pragma unroll 8
    for (int i = threadIdx.x; i < L; i += blockDim.x) dst[i] = src[i];
}

// exp(sign 2 pi i a / N) for 0 <= a < N = N1*N2 from two tables: twN2[i] = exp(-2 pi i i/N2)
// = exp(-2 pi i (N1 i)/N) and twF[i] = exp(-2 pi i i / N), i < N1.
template <int SIGN>
__device__ __forceinline__ C twiddleN(int a, int N1, const C* __restrict__ twN2, const C* __restrict__ twF) {
    C w = cmul(__ldg(&twN2[a / N1]), __ldg(&twF[a % N1]));
    return SIGN > 0 ? cconj(w) : w;
}

// u[idx] for idx < m: read directly, or summed from the per-cell scatter moments
// Mc[l][c + 2] (d = 1, rows of length m + 4): u[i] = Mc[0][i+3] + Mc[1][i+2] + Mc[2][i+1] + Mc[3][i]
__device__ __forceinline__ double u_at(const double* __restrict__ u, const double* __restrict__ Mc, int m, int idx) {
    if (Mc == nullptr) return u[idx];
    const int ld = m + 4;
    return Mc[idx + 3] + Mc[ld + idx + 2] + Mc[2 * ld + idx + 1] + Mc[3 * ld + idx];
}

// ---- single-CTA convolution (mode 0) / forward transform (mode 1), N <= 4096
template <int EPT>
__global__ void fft_small_kernel(const double* __restrict__ u, const double* __restrict__ Mc, int m, int N,
                                 const C* __restrict__ tw, const double* __restrict__ lam, double* __restrict__ z,
                                 C* __restrict__ outc, int mode, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(kTrFft0, done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N;
    load_tw(tws, tw, N);
    double lv[EPT];                             // data-independent: loaded before the transform
#pragma unroll
    for (int e = 0; e < EPT; ++e) lv[e] = mode == 1 ? 0.0 : __ldg(&lam[threadIdx.x + e * blockDim.x]);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int i = threadIdx.x + e * blockDim.x;
        buf[pad(i)] = make_double2(i < m ? u_at(u, Mc, m, i) : 0.0, 0.0);
    }
    __syncthreads();
    if (EPT == 4) line_fft4<-1>(buf, N, tws);
    else line_fft<-1>(buf, N, tws);
    if (mode == 1) {
        #pragma unroll 8
        for (int i = threadIdx.x; i < N; i += blockDim.x) outc[i] = buf[pad(i)];
        return;
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int i = threadIdx.x + e * blockDim.x;
        buf[pad(i)].x *= lv[e];
        buf[pad(i)].y *= lv[e];
    }
    __syncthreads();
    if (EPT == 4) line_fft4<+1>(buf, N, tws);
    else line_fft<+1>(buf, N, tws);
    #pragma unroll 8
    for (int i = threadIdx.x; i < m; i += blockDim.x) z[i] = buf[pad(i)].x;
}

// ---- four-step pass A: for each n1, FFT over n2 of x[n1 + N1 n2], times w_N^{n1 k2}
template <int G, int EPT>
__global__ void fft_passA_kernel(const double* __restrict__ u, const double* __restrict__ Mc, int m, int N1, int N2,
                                 const C* __restrict__ tw2, const C* __restrict__ twF, C* __restrict__ Y, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(kTrFft0, done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N2;
    load_tw(tws, tw2, N2);
    const int n1_0 = blockIdx.x * G;
    const int N = N1 * N2;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t % G, n2 = t / G;
        const int idx = n1_0 + g + N1 * n2;
        buf[pad(g * N2 + n2)] = make_double2(idx < m ? u_at(u, Mc, m, idx) : 0.0, 0.0);
    }
    __syncthreads();
    if (EPT == 4) line_fft4<-1>(buf, N2, tws);
    else line_fft<-1>(buf, N2, tws);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N2, k2 = t % N2;
        const int n1 = n1_0 + g;
        Y[(int64_t)n1 * N2 + k2] = cmul(buf[pad(t)], twiddleN<-1>((n1 * k2) & (N - 1), N1, tw2, twF));
    }
}

// ---- four-step pass B: for each k2, FFT over n1 -> X[N2 k1 + k2];
// mode 0: times lamB[k2*N1 + k1], inverse FFT over k1, times w_N^{-n1 k2}, store back
// mode 1: store X in natural order into outc
template <int G, int EPT>
__global__ void fft_passB_kernel(C* __restrict__ Y, int N1, int N2, const C* __restrict__ tw1,
                                 const C* __restrict__ tw2, const C* __restrict__ twF,
                                 const double* __restrict__ lamB, C* __restrict__ outc, int mode, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(kTrFft1, done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N1;
    load_tw(tws, tw1, N1);
    const int k2_0 = blockIdx.x * G;
    const int N = N1 * N2;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t % G, n1 = t / G;
        buf[pad(g * N1 + n1)] = Y[(int64_t)n1 * N2 + k2_0 + g];
    }
    __syncthreads();
    if (EPT == 4) line_fft4<-1>(buf, N1, tws);
    else line_fft<-1>(buf, N1, tws);
    if (mode == 1) {
    #pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
            const int g = t % G, k1 = t / G;
            outc[(int64_t)N2 * k1 + k2_0 + g] = buf[pad(g * N1 + k1)];
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N1, k1 = t % N1;
        const double l = lamB[(int64_t)(k2_0 + g) * N1 + k1];
        buf[pad(t)].x *= l;
        buf[pad(t)].y *= l;
    }
    __syncthreads();
    if (EPT == 4) line_fft4<+1>(buf, N1, tws);
    else line_fft<+1>(buf, N1, tws);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t % G, n1 = t / G;
        const int k2 = k2_0 + g;
        Y[(int64_t)n1 * N2 + k2] = cmul(buf[pad(g * N1 + n1)], twiddleN<+1>((n1 * k2) & (N - 1), N1, tw2, twF));
    }
}

// ---- four-step pass C: for each n1, inverse FFT over k2; z[n1 + N1 n2] = Re(.)
template <int G, int EPT>
__global__ void fft_passC_kernel(const C* __restrict__ Y, int m, int N1, int N2, const C* __restrict__ tw2,
                                 double* __restrict__ z, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(kTrFft2, done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N2;
    load_tw(tws, tw2, N2);
    const int n1_0 = blockIdx.x * G;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N2, k2 = t % N2;
        buf[pad(t)] = Y[(int64_t)(n1_0 + g) * N2 + k2];
    }
    __syncthreads();
    if (EPT == 4) line_fft4<+1>(buf, N2, tws);
    else line_fft<+1>(buf, N2, tws);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {             // exactly EPT elements per thread
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t % G, n2 = t / G;
        const int idx = n1_0 + g + N1 * n2;
        if (idx < m) z[idx] = buf[pad(g * N2 + n2)].x;
    }
}

// ---- real-input convolution at half length (d = 1, N > kSmallFFT).  u is real and so is z,
// so the length-N circulant product runs on N' = N/2 complex points:
//   zeta[n] = u[2n] + i u[2n+1]            (pass A', four-step N' = N1' N2')
//   Z = FFT_N'(zeta);  E[K] = (Z[K] + conj Z[N'-K]) / 2,  O[K] = (Z[K] - conj Z[N'-K]) / 2i
//   X[K] = E[K] + w^K O[K],  X[K+N'] = E[K] - w^K O[K]            (w = exp(-2 pi i / N))
//   Y = lambda X (lambda real, symmetric, * s^2/N);  W[K] = (Y[K] + Y[K+N']) + i w^-K (Y[K] - Y[K+N'])
//   IFFT_N'(W)[n] = z[2n] + i z[2n+1]                                 (passes B' and C')
// Pass B' holds the line pair {k2, N2'-k2} (k2 = 0 pairs with N2'/2), so every partner
// index N' - K of its elements is in the CTA.

// pass A': for each n1, FFT over n2 of zeta[n1 + N1 n2], times w_N'^{n1 k2}
template <int G>
__global__ void rfft_passA_kernel(const double* __restrict__ u, const double* __restrict__ Mc, int m, int N1, int N2,
                                  const C* __restrict__ tw2, const C* __restrict__ twF, C* __restrict__ Y, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(kTrFft0, done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N2;
    const int n1_0 = blockIdx.x * G;
    const int Np = N1 * N2;
    C ow[8];                                    // output twiddles, loaded before the transform
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        ow[e] = twiddleN<-1>(((n1_0 + t / N2) * (t % N2)) & (Np - 1), N1, tw2, twF);
    }
    load_tw(tws, tw2, N2);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t % G, n2 = t / G;
        const int n = n1_0 + g + N1 * n2;
        const double re = 2 * n < m ? u_at(u, Mc, m, 2 * n) : 0.0;
        const double im = 2 * n + 1 < m ? u_at(u, Mc, m, 2 * n + 1) : 0.0;
        buf[pad(g * N2 + n2)] = make_double2(re, im);
    }
    __syncthreads();
    line_fft<-1>(buf, N2, tws);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N2, k2 = t % N2;
        Y[(int64_t)(n1_0 + g) * N2 + k2] = cmul(buf[pad(t)], ow[e]);
    }
}

// pass B': lines {ka, kb} of length N1 (64 threads, 8 elements each): FFT over n1, untangle
// and multiply by lambda, re-tangle, inverse FFT over k1, times w_N'^{-n1 k2}.
//   twU1[k1] = w_N^{N2 k1}, twU2[k2] = w_N^{k2}  (so w_N^K = twU1[k1] twU2[k2] for K = N2 k1 + k2)
//   lamN[K] = lambda[K] * s^2 / N for K = 0..N'
__global__ void rfft_passB_kernel(C* __restrict__ Y, int N1, int N2, const C* __restrict__ tw1,
                                  const C* __restrict__ tw2, const C* __restrict__ twF, const C* __restrict__ twU1,
                                  const C* __restrict__ twU2, const double* __restrict__ lamN, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(kTrFft1, done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N1;
    const int b = blockIdx.x;
    const int kl[2] = {b == 0 ? 0 : b, b == 0 ? N2 / 2 : N2 - b};
    const int Np = N1 * N2;
    // element e of this thread: line g = t / N1, position t % N1 (k1 in the middle, n1 at the
    // ends).  Its untangle twiddle, lambdas and output twiddle do not depend on the data: load
    // them first, so their latency overlaps the input loads and the forward transform.
    C uw[8], ow[8];
    double l1v[8], l2v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N1, x = t % N1;
        const int k2 = kl[g];
        uw[e] = cmul(__ldg(&twU1[x]), __ldg(&twU2[k2]));
        const int K = N2 * x + k2;
        l1v[e] = __ldg(&lamN[K]);
        l2v[e] = __ldg(&lamN[Np - K]);
        ow[e] = twiddleN<+1>((x * k2) & (Np - 1), N1, tw2, twF);
    }
    load_tw(tws, tw1, N1);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N1, n1 = t % N1;
        buf[pad(t)] = Y[(int64_t)n1 * N2 + kl[g]];
    }
    __syncthreads();
    line_fft<-1>(buf, N1, tws);
    C wv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N1, k1 = t % N1;
        const int k2 = kl[g];
        int gp, k1p;                                   // partner of K = N2 k1 + k2: N' - K (mod N')
        if (k2 == 0) { gp = g; k1p = (N1 - k1) & (N1 - 1); }
        else if (2 * k2 == N2) { gp = g; k1p = N1 - 1 - k1; }
        else { gp = 1 - g; k1p = N1 - 1 - k1; }
        const C zk = buf[pad(t)];
        const C zq = cconj(buf[pad(gp * N1 + k1p)]);
        const C E = make_double2(0.5 * (zk.x + zq.x), 0.5 * (zk.y + zq.y));
        const C D = make_double2(0.5 * (zk.x - zq.x), 0.5 * (zk.y - zq.y));   // O = -i D
        const C O = make_double2(D.y, -D.x);
        const C w = uw[e];
        const C wO = cmul(w, O);
        const double l1 = l1v[e], l2 = l2v[e];          // lambda[K + N'] = lambda[N' - K]
        const C Y1 = make_double2(l1 * (E.x + wO.x), l1 * (E.y + wO.y));
        const C Y2 = make_double2(l2 * (E.x - wO.x), l2 * (E.y - wO.y));
        const C S = cadd(Y1, Y2);
        const C Dm = cmul(cconj(w), csub(Y1, Y2));
        wv[e] = make_double2(S.x - Dm.y, S.y + Dm.x);   // S + i Dm
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 8; ++e) buf[pad(threadIdx.x + e * blockDim.x)] = wv[e];
    __syncthreads();
    line_fft<+1>(buf, N1, tws);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N1, n1 = t % N1;
        Y[(int64_t)n1 * N2 + kl[g]] = cmul(buf[pad(t)], ow[e]);
    }
}

// pass C': for each n1, inverse FFT over k2; z[2n] = Re, z[2n+1] = Im at n = n1 + N1 n2
template <int G>
__global__ void rfft_passC_kernel(const C* __restrict__ Y, int m, int N1, int N2, const C* __restrict__ tw2,
                                  double* __restrict__ z, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(kTrFft2, done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N2;
    load_tw(tws, tw2, N2);
    const int n1_0 = blockIdx.x * G;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t / N2, k2 = t % N2;
        buf[pad(t)] = Y[(int64_t)(n1_0 + g) * N2 + k2];
    }
    __syncthreads();
    line_fft<+1>(buf, N2, tws);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int g = t % G, n2 = t / G;
        const int n = n1_0 + g + N1 * n2;
        const C w = buf[pad(g * N2 + n2)];
        if (2 * n < m) z[2 * n] = w.x;
        if (2 * n + 1 < m) z[2 * n + 1] = w.y;
    }
}

__global__ void lambda_natural_kernel(const C* __restrict__ X, int count, double scale, double* __restrict__ lamN) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) lamN[k] = X[k].x * scale;
}

// ---- dense per-axis Toeplitz products on the FP64 tensor cores (d > 1; K_UU is the
// Kronecker product of the per-axis Toeplitz T(c_d), applied axis by axis).  Along axis d the
// data [O][L][I] is the matrix X (L x O*I) and the axis product is D = T X, a GEMM with
// K = L: a CTA computes a 64 (rows r) x NT (columns) tile with mma.sync m8n8k4 f64 (DMMA),
// the whole K range of X staged once in shared memory (column-major by K), T's fragments read
// from the column c_d (T[r][k] = c_d[|r - k|]).  Warp w owns rows 8w .. 8w+7 and the NT / 8
// column tiles (independent accumulator chains).  LFAST (I == 1, the last axis): the columns
// are the lines (X[l][n] = in[n L + l]).  The tile goes out through shared memory, coalesced.
// fp64 throughout (products and sums), like the FFT path it replaces; only the order of the
// sums differs.
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// T3 != nullptr (first axis of a 3-D grid, LOVE_FUSE_PULL3): the X tile is the scatter's node
// sums u = s_j sum_a sum_b T3[a*4 + b][x + (1 - a) s0 + (1 - b) s1] formed on the fly from the
// fp32 last-axis sums (pull_mid_first_kernel's order: bitwise the same u), so u never goes
// through global memory and the pull_mid_first launch goes away
template <bool LFAST, int NT, bool MMA>
__global__ void __launch_bounds__(256) axis_mma_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                       const double* __restrict__ col, int L, int I, int64_t O,
                                                       double scale, const int* __restrict__ done,
                                                       const float* __restrict__ T3, int m1, int m2, StepRef ref3) {
    pdl_wait();
    LOVE_TRACE(LFAST ? kTrFft2 : (O == 1 ? kTrFft0 : kTrFft1), done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    constexpr int LD = NT + 1;                  // shared-memory row stride (doubles)
    extern __shared__ __align__(16) double smx[];
    double* cs = smx;                           // [L]    c_d
    double* Xs = smx + L;                       // [L][LD] X tile, then the [64][LD] D tile
    const int64_t n0 = (int64_t)blockIdx.x * NT;
    const int rb = blockIdx.y * 64;
    int64_t o = 0;
    int i0 = 0;
    if (!LFAST) {
        o = n0 / I;
        i0 = (int)(n0 - o * I);
    }
    for (int e = threadIdx.x; e < L; e += blockDim.x) cs[e] = col[e];
    if (LFAST) {
        for (int e = threadIdx.x; e < NT * L; e += blockDim.x) {
            const int n = e / L, l = e - n * L;
            Xs[l * LD + n] = n0 + n < O ? in[(n0 + n) * L + l] : 0.0;
        }
    } else if (T3 != nullptr) {
        const int64_t m = (int64_t)L * I;
        const double sj = ref3.scale[step_j(ref3)];
        for (int e = threadIdx.x; e < NT * L; e += blockDim.x) {
            const int l = e / NT, n = e - l * NT;
            const int64_t x = (int64_t)l * I + i0 + n;
            const int i1 = ((i0 + n) / m2) % m1;
            double sum = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int c0 = l - a + 1;
                if (c0 < 0 || c0 >= L) continue;
                const int64_t xa = x + (int64_t)(1 - a) * I;
                double va = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int c1 = i1 - b + 1;
                    if (c1 < 0 || c1 >= m1) continue;
                    va += (double)T3[(int64_t)(a * 4 + b) * m + xa + (1 - b) * m2];
                }
                sum += va;
            }
            Xs[l * LD + n] = sum * sj;
        }
    } else {
        for (int e = threadIdx.x; e < NT * L; e += blockDim.x) {
            const int l = e / NT, n = e - l * NT;
            Xs[l * LD + n] = in[(o * L + l) * (int64_t)I + i0 + n];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* Ds = Xs;                            // [64][LD], after the X tile is consumed
    if constexpr (MMA) {
        const int ra = rb + w * 8 + (lane >> 2);    // A fragment row
        const int ka = lane & 3;                    // A fragment column / B fragment row
        const int nb = lane >> 2;                   // B fragment column
        constexpr int NTT = NT / 8;
        double acc[NTT][2];
#pragma unroll
        for (int t = 0; t < NTT; ++t) acc[t][0] = acc[t][1] = 0.0;
        for (int k0 = 0; k0 < L; k0 += 4) {
            const int dk = ra - (k0 + ka);
            const double a = cs[dk < 0 ? -dk : dk];
            const double* xr = Xs + (k0 + ka) * LD + nb;
#pragma unroll
            for (int t = 0; t < NTT; ++t) dmma_8x8x4(acc[t], a, xr[t * 8]);
        }
        __syncthreads();                            // every warp is done with the X tile
#pragma unroll
        for (int t = 0; t < NTT; ++t) {
            const int r = w * 8 + (lane >> 2), n = t * 8 + (lane & 3) * 2;
            Ds[r * LD + n] = acc[t][0] * scale;
            Ds[r * LD + n + 1] = acc[t][1] * scale;
        }
    } else {
        // SIMT fp64: warp w owns rows 8w .. 8w+7, lane (n < NT) one column; c_d entries are
        // warp-uniform (broadcast), the X entry one conflict-free load per k
        constexpr int CPL = NT / 32 > 0 ? NT / 32 : 1;
        const bool live = lane < NT;
        double acc[8][CPL];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int q = 0; q < CPL; ++q) acc[u][q] = 0.0;
        const int r0 = rb + w * 8;
        for (int k = 0; k < L; ++k) {
            double x[CPL];
#pragma unroll
            for (int q = 0; q < CPL; ++q) x[q] = live ? Xs[k * LD + lane + 32 * q] : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int dk = r0 + u - k;
                const double cv = cs[dk < 0 ? -dk : dk];
#pragma unroll
                for (int q = 0; q < CPL; ++q) acc[u][q] = fma(cv, x[q], acc[u][q]);
            }
        }
        __syncthreads();
        if (live)
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int q = 0; q < CPL; ++q) Ds[(w * 8 + u) * LD + lane + 32 * q] = acc[u][q] * scale;
    }
    __syncthreads();
    if (LFAST) {
        for (int e = threadIdx.x; e < NT * 64; e += blockDim.x) {
            const int n = e / 64, r = e - n * 64;
            if (n0 + n < O) out[(n0 + n) * L + rb + r] = Ds[r * LD + n];
        }
    } else {
        for (int e = threadIdx.x; e < 64 * NT; e += blockDim.x) {
            const int r = e / NT, n = e - r * NT;
            out[(o * L + rb + r) * (int64_t)I + i0 + n] = Ds[r * LD + n];
        }
    }
}

// ---- dense per-axis Toeplitz products (d > 1), fp64
// layout (outer O, length L, inner I): out(o,l,i) = scale * sum_l' c[|l-l'|] in(o,l',i).
// Strided axes (I > 1): a CTA computes a 16 (rows) x 32 (inner) output tile, looping over
// 32-row chunks of the input staged in shared memory; 4 independent accumulators/thread.
constexpr int kAxRows = 16, kAxInner = 32, kAxK = 32;
__global__ void __launch_bounds__(128) axis_inner_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                         const double* __restrict__ c, int L, int I, double scale, const int* __restrict__ done) {
    pdl_wait();
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    __shared__ double cs[1024];
    __shared__ double tile[kAxK][kAxInner + 1];
    const int i0 = blockIdx.x * kAxInner;
    const int r0 = blockIdx.y * kAxRows;
    const int64_t ob = (int64_t)blockIdx.z * L * I;
    #pragma unroll 8
    for (int t = threadIdx.x; t < L; t += blockDim.x) cs[t] = c[t];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // 4 row groups of 4 rows
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int l0 = 0; l0 < L; l0 += kAxK) {
        __syncthreads();
        #pragma unroll 8
        for (int t = threadIdx.x; t < kAxK * kAxInner; t += blockDim.x) {
            const int l = t >> 5, ii = t & 31;
            tile[l][ii] = (l0 + l < L && i0 + ii < I) ? in[ob + (int64_t)(l0 + l) * I + i0 + ii] : 0.0;
        }
        __syncthreads();
        const int lmax = min(kAxK, L - l0);
        for (int l = 0; l < lmax; ++l) {
            const double v = tile[l][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = r0 + ty * 4 + q;
                acc[q] += cs[abs(r - (l0 + l)) & 1023] * v;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int r = r0 + ty * 4 + q;
        if (r < L && i0 + tx < I) out[ob + (int64_t)r * I + i0 + tx] = acc[q] * scale;
    }
}

// Contiguous axis (I = 1): one output per thread, 256 outputs per CTA (256/L lines, or a
// 256-row slice of one line), 4 partial sums per output.
__global__ void __launch_bounds__(256) axis_line_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                        const double* __restrict__ c, int64_t O, int L,
                                                        double scale, const int* __restrict__ done) {
    pdl_wait();
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    __shared__ double cs[1024];
    __shared__ double lines[2 * 1024 + 256];
    const int64_t first = (int64_t)blockIdx.x * 256;           // first output of this CTA
    const int64_t o0 = first / L;
    const int span = 2 * L + 256;                               // covers every line the CTA touches
    #pragma unroll 8
    for (int t = threadIdx.x; t < L; t += blockDim.x) cs[t] = c[t];
    #pragma unroll 8
    for (int t = threadIdx.x; t < span; t += blockDim.x) {
        const int64_t e = o0 * L + t;
        lines[t] = e < O * L ? in[e] : 0.0;
    }
    __syncthreads();
    const int64_t o = first + threadIdx.x;
    if (o >= O * L) return;
    const int ln = (int)(o / L - o0), r = (int)(o % L);
    const double* x = lines + ln * L;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int l = 0;
    for (; l + 4 <= L; l += 4) {
        a0 += cs[abs(r - l)] * x[l];
        a1 += cs[abs(r - l - 1)] * x[l + 1];
        a2 += cs[abs(r - l - 2)] * x[l + 2];
        a3 += cs[abs(r - l - 3)] * x[l + 3];
    }
    for (; l < L; ++l) a0 += cs[abs(r - l)] * x[l];
    out[o] = ((a0 + a1) + (a2 + a3)) * scale;
}

// ---- d > 1: T(c_d) applied along axis d by circulant-embedding FFTs of length N_d (P:187-188,
// reading A25), batched over the lines of the axis.  lambda_d is real and symmetric, so the
// circulant maps real lines to real lines and two lines travel as one complex line
// (x1 + i x2 -> T x1 + i T x2).  Data viewed as [O][L][I]; line (o, i) = in[(o L + l) I + i].
// P complex lines per CTA, P*N/8 threads (radix-8 Stockham, 8 elements per thread).
// LFAST (I == 1): a pair is two consecutive lines (o, o+1) and threads walk along l;
// otherwise a pair is (i, i+1) of one o and threads walk across pairs (coalesced in i).
template <bool LFAST, int EPT>
__global__ void axis_conv_kernel(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ lam,
                                 const C* __restrict__ tw, int L, int I, int64_t O, int N, int P, int64_t npairs,
                                 double scale, const int* __restrict__ done) {
    pdl_wait();
    LOVE_TRACE(O == 1 ? kTrFft0 : (LFAST ? kTrFft2 : kTrFft1), done != nullptr ? done[4] : 0);
    if (done != nullptr && *done) return;       // the Lanczos has stopped (breakdown or k)
    extern __shared__ __align__(16) unsigned char smraw[];
    C* tws = (C*)smraw;
    C* buf = tws + N;
    load_tw(tws, tw, N);
    const int64_t q0 = (int64_t)blockIdx.x * P;
    const int halfI = (I + 1) / 2;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int p = LFAST ? t / N : t % P, n = LFAST ? t % N : t / P;
        const int64_t q = q0 + p;
        double x1 = 0.0, x2 = 0.0;
        if (q < npairs && n < L) {
            if (LFAST) {
                const int64_t o = 2 * q;
                x1 = in[o * L + n];
                if (o + 1 < O) x2 = in[(o + 1) * L + n];
            } else {
                const int64_t o = q / halfI;
                const int i = 2 * (int)(q - o * halfI);
                const int64_t base = (o * L + n) * I + i;
                x1 = in[base];
                if (i + 1 < I) x2 = in[base + 1];
            }
        }
        buf[pad(p * N + n)] = make_double2(x1, x2);
    }
    double lv[EPT];                              // data-independent: loaded before the transform
#pragma unroll
    for (int e = 0; e < EPT; ++e) lv[e] = __ldg(&lam[(threadIdx.x + e * blockDim.x) % N]);
    __syncthreads();
    if (EPT == 4) line_fft4<-1>(buf, N, tws);
    else line_fft<-1>(buf, N, tws);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        buf[pad(t)].x *= lv[e];
        buf[pad(t)].y *= lv[e];
    }
    __syncthreads();
    if (EPT == 4) line_fft4<+1>(buf, N, tws);
    else line_fft<+1>(buf, N, tws);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int t = threadIdx.x + e * blockDim.x;
        const int p = LFAST ? t / N : t % P, n = LFAST ? t % N : t / P;
        const int64_t q = q0 + p;
        if (q >= npairs || n >= L) continue;
        const C v = buf[pad(p * N + n)];
        if (LFAST) {
            const int64_t o = 2 * q;
            out[o * L + n] = v.x * scale;
            if (o + 1 < O) out[(o + 1) * L + n] = v.y * scale;
        } else {
            const int64_t o = q / halfI;
            const int i = 2 * (int)(q - o * halfI);
            const int64_t base = (o * L + n) * I + i;
            out[base] = v.x * scale;
            if (i + 1 < I) out[base + 1] = v.y * scale;
        }
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

__global__ void twiddle_table_kernel(C* __restrict__ tw, int L, int den) {
    // tw[k] = exp(-2 pi i k / den), k < L
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < L; k += gridDim.x * blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)k / (double)den, &s, &c);
        tw[k] = make_double2(c, -s);
    }
}

__global__ void embed_kernel(const double* __restrict__ c, int m, int N, double* __restrict__ col) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const int a = min(i, N - i);            // circulant distance (N >= 2m - 1: i < m or i > N - m)
        col[i] = a < m ? c[a] : 0.0;
    }
}

__global__ void lambda_store_kernel(const C* __restrict__ X, int N, int N1, int N2, int four_step,
                                    double scale, double* __restrict__ lam) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        const double v = X[k].x * scale;
        if (four_step) {
            const int k1 = k / N2, k2 = k % N2;   // k = N2 k1 + k2
            lam[(int64_t)k2 * N1 + k1] = v;
        } else {
            lam[k] = v;
        }
    }
}

inline int ilog2(int64_t x) {
    int l = 0;
    while ((int64_t(1) << l) < x) ++l;
    return l;
}

constexpr int kSmallFFT = 4096;

// convolution (mode 0) of u (m entries) or forward FFT (mode 1) of u (N entries)
// complex four-step passes: GA columns per CTA in passes A / C, GB lines per CTA in pass B
template <int GA, int GB, int EPT>
static void fft_four_step(const Cache& c, const double* u, const double* Mc, int m, double* z, C* work, C* outc,
                          int mode, cudaStream_t s) {
    const int N1 = c.fft_N1, N2 = c.fft_N2;
    const C* tw1 = (const C*)c.tw1;
    const C* tw2 = (const C*)c.tw2;
    const C* twF = (const C*)c.twF;
    const double* lam = (const double*)c.lam;
    const size_t smA = sizeof(C) * (padded((size_t)GA * N2) + N2), smB = sizeof(C) * (padded((size_t)GB * N1) + N1);
    ensure_smem((const void*)fft_passA_kernel<GA, EPT>, smA);
    ensure_smem((const void*)fft_passB_kernel<GB, EPT>, smB);
    ensure_smem((const void*)fft_passC_kernel<GA, EPT>, smA);
    LOVE_LAUNCH((fft_passA_kernel<GA, EPT>), N1 / GA, GA * N2 / EPT, smA, s, u, Mc, m, N1, N2, tw2, twF, work, t_done);
    LOVE_LAUNCH((fft_passB_kernel<GB, EPT>), N2 / GB, GB * N1 / EPT, smB, s, work, N1, N2, tw1, tw2, twF, lam, outc,
                mode, t_done);
    if (mode == 0)
        LOVE_LAUNCH((fft_passC_kernel<GA, EPT>), N1 / GA, GA * N2 / EPT, smA, s, (const C*)work, m, N1, N2, tw2, z,
                    t_done);
}

// measurement switches: LOVE_FFT_GA / LOVE_FFT_GB (lines per CTA, EPT = 4 convolution only)
template <int EPT>
static bool fft_four_step_env(const Cache& c, const double* u, const double* Mc, int m, double* z, C* work, C* outc,
                              int mode, cudaStream_t s) {
    static const int ga = std::getenv("LOVE_FFT_GA") ? std::atoi(std::getenv("LOVE_FFT_GA")) : 0;
    static const int gb = std::getenv("LOVE_FFT_GB") ? std::atoi(std::getenv("LOVE_FFT_GB")) : 0;
    if (ga == 0 || gb == 0 || mode != 0 || EPT != 4) return false;
#define LOVE_FS(A_, B_) \
    if (ga == A_ && gb == B_) { fft_four_step<A_, B_, EPT>(c, u, Mc, m, z, work, outc, mode, s); return true; }
    LOVE_FS(1, 1) LOVE_FS(1, 2) LOVE_FS(1, 4) LOVE_FS(2, 1) LOVE_FS(2, 2) LOVE_FS(2, 4) LOVE_FS(4, 1) LOVE_FS(4, 2)
    LOVE_FS(4, 4) LOVE_FS(8, 1) LOVE_FS(8, 2) LOVE_FS(8, 4) LOVE_FS(16, 1) LOVE_FS(16, 2)
#undef LOVE_FS
    return false;
}

void fft_run(const Cache& c, const double* u, const double* Mc, int m, double* z, C* work, C* outc, int mode,
             cudaStream_t s) {
    const int N = c.fft_N, N1 = c.fft_N1;
    const C* tw1 = (const C*)c.tw1;
    const double* lam = (const double*)c.lam;
    if (N1 == 0) {
        const size_t sm = sizeof(C) * (padded(N) + N);
        static const int ept = std::getenv("LOVE_FFT_EPT") ? std::atoi(std::getenv("LOVE_FFT_EPT")) : 4;
        if (ept == 4 && mode == 0 && N >= 8 && N / 4 <= 1024) {
            ensure_smem((const void*)fft_small_kernel<4>, sm);
            LOVE_LAUNCH(fft_small_kernel<4>, 1, N / 4, sm, s, u, Mc, m, N, tw1, lam, z, outc, mode, t_done);
        } else {
            ensure_smem((const void*)fft_small_kernel<8>, sm);
            LOVE_LAUNCH(fft_small_kernel<8>, 1, std::max(1, N / 8), sm, s, u, Mc, m, N, tw1, lam, z, outc, mode,
                        t_done);
        }
        return;
    }
    constexpr int G = 2;
    if (mode == 0 && c.rfft_N1 != 0) {          // real-input half-length convolution
        const int R1 = c.rfft_N1, R2 = c.rfft_N2;
        const C* r1 = (const C*)c.rtw1;
        const C* r2 = (const C*)c.rtw2;
        const C* rF = (const C*)c.rtwF;
        const size_t sA = sizeof(C) * (padded((size_t)G * R2) + R2), sB = sizeof(C) * (padded((size_t)2 * R1) + R1);
        ensure_smem((const void*)rfft_passA_kernel<G>, sA);
        ensure_smem((const void*)rfft_passB_kernel, sB);
        ensure_smem((const void*)rfft_passC_kernel<G>, sA);
        LOVE_LAUNCH(rfft_passA_kernel<G>, R1 / G, G * R2 / 8, sA, s, u, Mc, m, R1, R2, r2, rF, work, t_done);
        LOVE_LAUNCH(rfft_passB_kernel, R2 / 2, 2 * R1 / 8, sB, s, work, R1, R2, r1, r2, rF, (const C*)c.rtwU1,
                    (const C*)c.rtwU2, (const double*)c.rlam, t_done);
        LOVE_LAUNCH(rfft_passC_kernel<G>, R1 / G, G * R2 / 8, sA, s, (const C*)work, m, R1, R2, r2, z, t_done);
        return;
    }
    // measured: 4 lines per CTA (16-byte loads in 64-byte runs) win at N <= 2^15 (cfg5 build
    // 6.11 -> 5.97 ms), 2 lines (twice the CTAs) at 2^17; 1 line loses everywhere
    // 4 elements per thread (radix-4 stages, twice the threads per CTA) for the convolution
    // passes of the Lanczos (LOVE_FFT_EPT=8: radix-8); the one-off forward transform of the
    // setup keeps radix 8
    static const int ept = std::getenv("LOVE_FFT_EPT") ? std::atoi(std::getenv("LOVE_FFT_EPT")) : 4;
    const bool e4 = ept == 4 && mode == 0;
    if (e4 && fft_four_step_env<4>(c, u, Mc, m, z, work, outc, mode, s)) return;
    if (N <= (1 << 15)) {
        if (e4) fft_four_step<4, 4, 4>(c, u, Mc, m, z, work, outc, mode, s);
        else fft_four_step<4, 4, 8>(c, u, Mc, m, z, work, outc, mode, s);
    } else {
        if (e4) fft_four_step<G, G, 4>(c, u, Mc, m, z, work, outc, mode, s);
        else fft_four_step<G, G, 8>(c, u, Mc, m, z, work, outc, mode, s);
    }
}

void kuu_axes(const Cache& c, const double* u, double* z, cudaStream_t s, const StepRef* pull3) {
    const GridDev& g = c.g;
    const double* in = u;
    int off = 0;
    for (int d = 0; d < g.d; ++d) {
        const int L = g.m[d];
        int O = 1, I = 1;
        for (int e = 0; e < d; ++e) O *= g.m[e];
        for (int e = d + 1; e < g.d; ++e) I *= g.m[e];
        double* out = (d == g.d - 1) ? z : (double*)c.ktmp[d & 1];
        const double scale = (d == g.d - 1) ? c.rbf.outputscale : 1.0;
        const double* col = c.cols64 + off;
        // FP64 tensor-core axis product for the short axes (L = 64; the shapes must tile: L a
        // multiple of 64 up to 512 (shared memory), I = 1 or a multiple of 32).  Measured in-graph: cfg4 (64^3) 9.5 -> 7.0 us per axis, build
        // 31.0 -> 30.2 ms; at L = 256 (cfg3) the FFT won with 32-column tiles (7.9 vs 8.7 ms) and
        // loses with 8-column ones (axis slots 8.0 + 6.9 -> 6.3 + 6.7 us, cfg3 7.69 -> 7.47 ms).
        // LOVE_AXIS_MMA (read per call): unset = auto (L <= 256), 0 = FFT, 1 = DMMA for every
        // L that tiles, 2 = SIMT fp64 (measured: as DMMA at cfg4, slower at cfg3)
        const char* mma_env = std::getenv("LOVE_AXIS_MMA");
        const int mma_mode = mma_env ? std::atoi(mma_env) : -1;
        const int64_t ncols = I == 1 ? (int64_t)O : (int64_t)O * I;
        if (mma_mode != 0 && (mma_mode > 0 || L <= 256) && L % 64 == 0 && L <= 512 && (I == 1 || I % 32 == 0)) {
            static const int nt_env = std::getenv("LOVE_AXIS_NT") ? std::atoi(std::getenv("LOVE_AXIS_NT")) : 0;
            // columns per CTA: halved from 32 while the grid has fewer than 4 CTAs per SM (measured
            // in-graph, cfg4: 128 CTAs of 32 columns 7.0 us per axis, 256 of 16 6.2 us, 512 of 8
            // 5.0 us; cfg4 28.62 -> 28.04 ms); LOVE_AXIS_NT = 8 / 16 / 32 overrides
            int NT = 32;
            while (NT > 8 && ncols / NT * (L / 64) < 4 * 148) NT /= 2;
            if (nt_env == 8 || nt_env == 16 || nt_env == 32) NT = nt_env;
            if (I != 1 && I % NT != 0) NT = 32;
            // the first axis of a 3-D grid can read the scatter's last-axis sums directly
            const bool from_t = pull3 != nullptr && d == 0 && g.d == 3 && I > 1;
            if (pull3 != nullptr && d == 0 && !from_t) throw LoveError{LOVE_ERR_CUDA, "fused pull: axis 0 not on DMMA"};
            const float* T3 = from_t ? (const float*)c.pullT : nullptr;
            const int m1v = g.m[1], m2v = g.m[2];
            const StepRef ref3 = from_t ? *pull3 : StepRef{nullptr, 0, nullptr, nullptr};
            const size_t sm = sizeof(double) * ((size_t)L + (size_t)std::max(L, 64) * (NT + 1));
            dim3 grid((unsigned)ceil_div(ncols, NT), (unsigned)(L / 64));
#define LOVE_AXMMA(LF, NT_)                                                                                  \
    do {                                                                                                     \
        if (mma_mode == 2) {                                                                                 \
            ensure_smem((const void*)axis_mma_kernel<LF, NT_, false>, sm);                                   \
            LOVE_LAUNCH((axis_mma_kernel<LF, NT_, false>), grid, 256, sm, s, in, out, col, L, I, (int64_t)O, scale, t_done, \
                        T3, m1v, m2v, ref3);                                                                 \
        } else {                                                                                             \
            ensure_smem((const void*)axis_mma_kernel<LF, NT_, true>, sm);                                    \
            LOVE_LAUNCH((axis_mma_kernel<LF, NT_, true>), grid, 256, sm, s, in, out, col, L, I, (int64_t)O, scale, t_done, \
                        T3, m1v, m2v, ref3);                                                                 \
        }                                                                                                    \
    } while (0)
            if (I == 1) {
                if (NT == 8) LOVE_AXMMA(true, 8);
                else if (NT == 16) LOVE_AXMMA(true, 16);
                else LOVE_AXMMA(true, 32);
            } else {
                if (NT == 8) LOVE_AXMMA(false, 8);
                else if (NT == 16) LOVE_AXMMA(false, 16);
                else LOVE_AXMMA(false, 32);
            }
#undef LOVE_AXMMA
        } else if (c.ax_N[d] > 0) {             // batched line FFTs (two real lines per complex line)
            const int N = c.ax_N[d];
            // complex lines per CTA: one for N >= 512 (cfg3, N = 512: twice the CTAs, half the
            // threads per barrier; 8.01 -> 7.84 ms against two), else 1024 / N (LOVE_AXIS_P overrides)
            const char* pe = std::getenv("LOVE_AXIS_P");
            const int P = pe ? std::max(1, std::min(8, std::atoi(pe)))
                             : (N >= 512 ? 1 : std::max(1, std::min(8, 1024 / N)));
            const int64_t npairs = I == 1 ? (O + 1) / 2 : (int64_t)O * ((I + 1) / 2);
            const size_t sm = sizeof(C) * (N + padded((size_t)P * N));
            const int grid = (int)ceil_div(npairs, P);
            // 4 elements per thread (radix-4) when the block stays <= 1024 threads (LOVE_AXIS_EPT=8: radix-8)
            static const int ept_env = std::getenv("LOVE_AXIS_EPT") ? std::atoi(std::getenv("LOVE_AXIS_EPT")) : 4;
            const bool e4 = ept_env == 4 && P * N / 4 <= 1024;
            const int thr = P * N / (e4 ? 4 : 8);
#define LOVE_AXIS_LAUNCH(LF, E)                                                                              \
    do {                                                                                                     \
        ensure_smem((const void*)axis_conv_kernel<LF, E>, sm);                                               \
        LOVE_LAUNCH((axis_conv_kernel<LF, E>), grid, thr, sm, s, in, out, (const double*)c.ax_lam[d],        \
                    (const C*)c.ax_tw[d], L, I, (int64_t)O, N, P, npairs, scale, t_done);                     \
    } while (0)
            if (I == 1) {
                if (e4) LOVE_AXIS_LAUNCH(true, 4);
                else LOVE_AXIS_LAUNCH(true, 8);
            } else {
                if (e4) LOVE_AXIS_LAUNCH(false, 4);
                else LOVE_AXIS_LAUNCH(false, 8);
            }
#undef LOVE_AXIS_LAUNCH
        } else if (I == 1) {
            const int64_t total = (int64_t)O * L;
            LOVE_LAUNCH(axis_line_kernel, (int)ceil_div(total, 256), 256, 0, s, in, out, col, (int64_t)O, L, scale, t_done);
        } else {
            dim3 grid((unsigned)ceil_div(I, kAxInner), (unsigned)ceil_div(L, kAxRows), (unsigned)O);
            LOVE_LAUNCH(axis_inner_kernel, grid, 128, 0, s, in, out, col, L, I, scale, t_done);
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
    LOVE_LAUNCH(rbf_columns_kernel, 64, 256, 0, s, g, c.rbf.lengthscale[0], c.rbf.lengthscale[1],
                c.rbf.lengthscale[2], c.cols64);
    for (int d = 0; d < g.d; ++d)     // c_d[0..3] on the host for the variance-query prior
        for (int i = 0; i < 4; ++i) {
            const double r = (double)i * g.h[d];
            c.h_cols64[d][i] = std::exp(-(r * r) / (2.0 * c.rbf.lengthscale[d] * c.rbf.lengthscale[d]));
        }
    if (g.d > 1) {
        for (int d = 0; d < g.d; ++d)
            if (g.m[d] > 1024) throw LoveError{LOVE_ERR_ARG, "Kronecker grids need m_d <= 1024 per axis"};
        c.ktmp[0] = dalloc(c, sizeof(double) * g.m_total, s);
        c.ktmp[1] = dalloc(c, sizeof(double) * g.m_total, s);
        // per-axis circulant eigenvalues lambda_d / N_d (FFT of the embedded column, mode 1)
        const bool use_fft = std::getenv("LOVE_AXIS_DENSE") == nullptr;
        int off = 0;
        for (int d = 0; d < g.d; ++d) {
            const int md = g.m[d];
            int Nd = 8;
            while (Nd < 2 * md - 1) Nd *= 2;
            c.ax_N[d] = 0;
            if (use_fft && Nd <= kSmallFFT) {
                c.ax_N[d] = Nd;
                c.ax_tw[d] = dalloc(c, sizeof(C) * Nd, s);
                c.ax_lam[d] = dalloc(c, sizeof(double) * Nd, s);
                LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(Nd, 256), 256, 0, s, (C*)c.ax_tw[d], Nd, Nd);
                double* colN = nullptr;
                C* X = nullptr;
                cuda_check(cudaMallocAsync((void**)&colN, sizeof(double) * Nd, s), "axis lam alloc");
                cuda_check(cudaMallocAsync((void**)&X, sizeof(C) * Nd, s), "axis lam alloc");
                LOVE_LAUNCH(embed_kernel, (int)ceil_div(Nd, 256), 256, 0, s, c.cols64 + off, md, Nd, colN);
                const size_t sm = sizeof(C) * (padded(Nd) + Nd);
                ensure_smem((const void*)fft_small_kernel<8>, sm);
                LOVE_LAUNCH(fft_small_kernel<8>, 1, std::max(1, Nd / 8), sm, s, colN, (const double*)nullptr, Nd, Nd,
                            (const C*)c.ax_tw[d], (const double*)nullptr, (double*)nullptr, X, 1, t_done);
                LOVE_LAUNCH(lambda_store_kernel, (int)ceil_div(Nd, 256), 256, 0, s, X, Nd, 0, 0, 0, 1.0 / (double)Nd,
                            (double*)c.ax_lam[d]);
                cuda_check(cudaFreeAsync(colN, s), "axis lam free");
                cuda_check(cudaFreeAsync(X, s), "axis lam free");
            }
            off += md;
        }
        return;
    }
    // d = 1: circulant embedding and its eigenvalues, stored * s^2 / N
    const int m = g.m[0];
    // Embedding length (reading A25b): the circulant of length N agrees with the
    // Toeplitz T(c) wherever the grid distance delta <= N/2; at delta > N/2 it holds c_{N-delta}
    // instead of c_delta.  N >= 2m - 1 makes that set empty.  When the RBF column
    // falls below 1e-30 c_0 from b = ceil(ls/h sqrt(2 ln 1e30)) on and b < m, N >= m + b is
    // enough: both c_{N-delta} (N - delta > b) and c_delta (delta > (m+b)/2 > b) are < 1e-30 c_0,
    // 14 orders below the fp64 rounding of the product.  cfg2: N = 2^17 instead of 2^18.
    int64_t need = 2 * (int64_t)m - 1;
    if (std::getenv("LOVE_FULL_EMBED") == nullptr) {
        const double b = std::ceil(std::sqrt(2.0 * std::log(1e30)) * c.rbf.lengthscale[0] / g.h[0]);
        if (b < (double)m) need = std::min<int64_t>(need, (int64_t)m + (int64_t)b);
    }
    int N = 8;
    while (N < need) N *= 2;
    if (N > (1 << 22)) throw LoveError{LOVE_ERR_ARG, "1-D grid too long (m <= 2^21)"};
    c.fft_N = N;
    if (N <= kSmallFFT) {
        c.fft_N1 = c.fft_N2 = 0;
        c.tw1 = dalloc(c, sizeof(C) * N, s);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(N, 256), 256, 0, s, (C*)c.tw1, N, N);
    } else {
        const int lg = ilog2(N);
        // N1 = 2^(lg/2) (LOVE_FFT_LG1: measurement switch)
        const int lg1 = std::getenv("LOVE_FFT_LG1") ? std::atoi(std::getenv("LOVE_FFT_LG1")) : lg / 2;
        c.fft_N1 = 1 << lg1;
        c.fft_N2 = N / c.fft_N1;
        c.tw1 = dalloc(c, sizeof(C) * c.fft_N1, s);
        c.tw2 = dalloc(c, sizeof(C) * c.fft_N2, s);
        c.twF = dalloc(c, sizeof(C) * c.fft_N1, s);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(c.fft_N1, 256), 256, 0, s, (C*)c.tw1, c.fft_N1, c.fft_N1);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(c.fft_N2, 256), 256, 0, s, (C*)c.tw2, c.fft_N2, c.fft_N2);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(c.fft_N1, 256), 256, 0, s, (C*)c.twF, c.fft_N1, N);
    }
    c.lam = dalloc(c, sizeof(double) * N, s);
    c.fft_buf = dalloc(c, sizeof(C) * N, s);
    double* col = nullptr;
    C* X = nullptr;
    cuda_check(cudaMallocAsync((void**)&col, sizeof(double) * N, s), "lam alloc");
    cuda_check(cudaMallocAsync((void**)&X, sizeof(C) * N, s), "lam alloc");
    LOVE_LAUNCH(embed_kernel, (int)std::min<int64_t>(ceil_div(N, 256), 4096), 256, 0, s, c.cols64, m, N, col);
    fft_run(c, col, nullptr, N, nullptr, (C*)c.fft_buf, X, 1, s);
    LOVE_LAUNCH(lambda_store_kernel, (int)std::min<int64_t>(ceil_div(N, 256), 4096), 256, 0, s, X, N, c.fft_N1,
                c.fft_N2, c.fft_N1 != 0, c.rbf.outputscale / (double)N, (double*)c.lam);
    // measured: the half-length real path wins at N = 2^18 but not at 2^17 (cfg2 with the
    // shortened embedding: 11.2 vs 11.4 ms per build) or 2^15: the passes are latency-bound and
    // half as many CTAs hide less of it
    // real-input half-length passes from N >= 2^18 (LOVE_RFFT_MIN = log2 of the threshold)
    const int rfft_min = std::getenv("LOVE_RFFT_MIN") ? std::atoi(std::getenv("LOVE_RFFT_MIN")) : 18;
    if (c.fft_N1 != 0 && N >= (1 << rfft_min) && std::getenv("LOVE_NO_RFFT") == nullptr) {
        // real-input path: N' = N/2 = R1 * R2 (R1 = 2^floor(lg N'/2)), tables and lambda[0..N']
        const int Np = N / 2, lgp = ilog2(Np);
        c.rfft_N1 = 1 << (lgp / 2);
        c.rfft_N2 = Np / c.rfft_N1;
        const int R1 = c.rfft_N1, R2 = c.rfft_N2;
        c.rtw1 = dalloc(c, sizeof(C) * R1, s);
        c.rtw2 = dalloc(c, sizeof(C) * R2, s);
        c.rtwF = dalloc(c, sizeof(C) * R1, s);
        c.rtwU1 = dalloc(c, sizeof(C) * R1, s);
        c.rtwU2 = dalloc(c, sizeof(C) * R2, s);
        c.rlam = dalloc(c, sizeof(double) * (Np + 1), s);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(R1, 256), 256, 0, s, (C*)c.rtw1, R1, R1);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(R2, 256), 256, 0, s, (C*)c.rtw2, R2, R2);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(R1, 256), 256, 0, s, (C*)c.rtwF, R1, Np);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(R1, 256), 256, 0, s, (C*)c.rtwU1, R1, 2 * R1);
        LOVE_LAUNCH(twiddle_table_kernel, (int)ceil_div(R2, 256), 256, 0, s, (C*)c.rtwU2, R2, N);
        LOVE_LAUNCH(lambda_natural_kernel, (int)std::min<int64_t>(ceil_div(Np + 1, 256), 4096), 256, 0, s, X, Np + 1,
                    c.rbf.outputscale / (double)N, (double*)c.rlam);
    }
    cuda_check(cudaFreeAsync(col, s), "lam free");
    cuda_check(cudaFreeAsync(X, s), "lam free");
}

bool fuse_pull3(const Cache& c) {
    static const bool on = std::getenv("LOVE_FUSE_PULL3") == nullptr || std::atoi(std::getenv("LOVE_FUSE_PULL3")) != 0;
    if (!on || c.additive || c.g.d != 3 || c.comm != nullptr || c.precision != LOVE_FP32 || c.fused) return false;
    if (std::getenv("LOVE_PULL_T64") != nullptr || std::getenv("LOVE_PULL_MF") != nullptr) return false;
    // the first axis must take the DMMA path (kuu_axes' rule)
    const char* mma_env = std::getenv("LOVE_AXIS_MMA");
    const int mma_mode = mma_env ? std::atoi(mma_env) : -1;
    const int L = c.g.m[0], I = c.g.m[1] * c.g.m[2];
    return mma_mode != 0 && (mma_mode > 0 || L <= 256) && L % 64 == 0 && L <= 512 && I % 32 == 0;
}

void launch_kuu(const Cache& c, const double* u, double* z, cudaStream_t s, const double* Mc, const StepRef* pull3) {
    if (c.additive) {
        add_kuu(c, u, z, s);
        return;
    }
    if (c.g.d > 1) kuu_axes(c, u, z, s, pull3);
    else fft_run(c, u, Mc, c.g.m[0], z, (C*)c.fft_buf, nullptr, 0, s);
}

}  // namespace love
