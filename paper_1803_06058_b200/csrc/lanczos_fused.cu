// lanczos_fused.cu -- one-read Lanczos (fp32 mode): the full reorthogonalisation of step j-1
// is applied lazily inside the single pass over the training points of step j.
//
// Classical scheme (lanczos.cu, P:139-150 + P:821): per step the Krylov basis Q_j is read
// twice (c = Q_j^T r', then q~ = r' - Q_j c).  Here both reads are the same read:
//
//  pass F_j over the points, tile by tile (one Q~ tile staged in shared memory):
//     r'_{j-1} = s_{j-1} r~_{j-1} - alpha_{j-1} q_{j-1} - beta_{j-2} q_{j-2}
//     Q~_j     = r'_{j-1} - sum_{i<j} c_{j-1,i} q_i          (lagged CGS update)
//     r~_j     = W^T z~_j + sigma^2 Q~_j                      (SKI MVM gather)
//     M        = stencil moments of r~_j                      (for the scatter W r~_j)
//     A_i = Q~_i . r~_j,  B_i = Q~_i . Q~_j    for i <= j     (Gram sums, fp64)
//  scalars:   beta_{j-1} = sqrt(B_j) = ||Q~_j||, s_j = 1/beta_{j-1}, alpha_j = s_j^2 A_j,
//             c_{j,i} = q_i^T r'_j from the Gram sums (no extra pass; SURVEY X9 one-sync form)
//  m side:    Rc[:, j], a  (streamed cache, as in lanczos.cu), and
//             u~_{j+1} = W Q~_{j+1} = s_j W r~_j - sum_i gamma_i u~_i   (linearity of W)
//             z~_{j+1} = K_UU u~_{j+1}
// so q_{j+1} is materialised only in pass F_{j+1}, yet its MVM is ready before that pass.
// Columns of Q~ are stored unnormalised (q_i = s_i Q~_i).  The u~_i are kept in fp64 for the
// two newest and in fp32 for the (tiny) reorthogonalisation correction.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "love_internal.h"
#include "ski_device.cuh"
#include "tma.cuh"

namespace love {

namespace {

constexpr int kZMax = 1280;           // staged z~ nodes per tile (d <= 2)

// 2-D tensor TMA: box {rows, 8 columns} of the column-major Q~ at coordinates (row, col)
__device__ __forceinline__ void tma_q_box(void* dst, const CUtensorMap* map, int row, int col, uint64_t* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(d), "l"(reinterpret_cast<uint64_t>(map)), "r"(row), "r"(col), "r"(b) : "memory");
}
constexpr int kBoxCols = 8;

// Per-tile descriptor, computed once per build (tile_meta_kernel): 12 ints, 48 bytes.
struct TileMeta {
    int it0, it1;        // items [it0, it1)
    int p0, p1;          // points [p0, p1)
    int a0, nch;         // 16-byte aligned first point, 16-byte chunks of every point array
    int zlo, zspan;      // staged z~ nodes [zlo, zlo + zspan) (zspan = 0: load z~ from global)
    int ia0, nich;       // 16-byte aligned first item, chunks of the staged item arrays
    int pad0, pad1;
};

struct FusedArgs {
    GridDev g;
    int64_t ldq, n_items, n_tiles;
    int k, RS, IS;                   // RS / IS: shared-memory strides of a staged point / item array
    float* Q;                        // [k+1][ldq] unnormalised Krylov columns
    float* rt;                       // r~: holds r~_{j-1} on entry, r~_j on exit
    const float *f0, *f1, *f2;       // sorted fractional offsets
    const int* item_cell;
    const int* item_start;
    const TileMeta* meta;
    const double* z;                 // z~_j (fp64), padded
    double sigma2;
    double* M;                       // [4^d][n_items] moments of r~_j
    double* M2;                      // [4^d][n_items] moments of Q~_j
    LanczosState st;
    int debug_mode;
};

// staging-buffer layout: [z~ nodes (d <= 2)][Q~ columns][r~_{j-1}][offsets][item_start][item_cell]
struct BufLayout {
    size_t qoff, roff, foff, ioff, coff, stride;
};
__host__ __device__ inline BufLayout buf_layout(int k, int RS, int IS, int d) {
    BufLayout L;
    L.qoff = d <= 2 ? sizeof(double) * kZMax : 0;                           // 128-B multiple
    L.roff = L.qoff + sizeof(float) * (size_t)(((k + 1 + 7) / 8) * 8) * RS;  // whole 8-column boxes
    L.foff = L.roff + sizeof(float) * RS;
    L.ioff = L.foff + sizeof(float) * (size_t)d * RS;
    L.coff = L.ioff + sizeof(int) * IS;
    L.stride = ((L.coff + sizeof(int) * IS + 127) / 128) * 128;            // buffers 128-B aligned
    return L;
}

// bytes of dynamic shared memory of the fused pass
size_t fused_smem(int k, int RS, int IS, int d) {
    const BufLayout L = buf_layout(k, RS, IS, d);
    const size_t wts = std::max<size_t>(4 * (size_t)d * RS, 2048);
    const size_t single = sizeof(double) * 2 * (k + 1) + sizeof(float) * (RS + wts) +
                          sizeof(int) * RS + sizeof(float) * round_up(k + 1, 4);
    return 128 + 2 * L.stride + single;
}

__device__ __forceinline__ TileMeta load_meta(const TileMeta* meta, int64_t t) {
    const int4* src = reinterpret_cast<const int4*>(meta + t);
    const int4 x = __ldg(src), y = __ldg(src + 1), w = __ldg(src + 2);
    return TileMeta{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w, w.x, w.y, w.z, w.w};
}

// warp 0: publish the tile descriptor and start the bulk copies of the tile into one buffer
template <int D>
__device__ void issue_tile(const FusedArgs& a, const CUtensorMap* qmap, int j, const TileMeta& mt, TileMeta* ti,
                           uint64_t* bar, unsigned char* bp, const BufLayout& L) {
    const int lane = threadIdx.x & 31;
    const unsigned cbytes = (unsigned)mt.nch * 16u, ibytes = (unsigned)mt.nich * 16u;
    const int ncopy = j >= 1 ? j : 1;
    const bool empty = mt.it1 <= mt.it0;
    if (lane == 0) {
        *ti = mt;
        if (empty) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar))
                         : "memory");
        } else {
            const unsigned nbox = (unsigned)((ncopy + kBoxCols - 1) / kBoxCols);
            const unsigned total = nbox * (unsigned)(kBoxCols * a.RS * 4) + cbytes * (unsigned)((j >= 1 ? 1 : 0) + D) +
                                   2u * ibytes + (unsigned)mt.zspan * 8u;
            mbar_expect_tx(bar, total);
        }
    }
    __syncwarp();
    if (empty) return;
    const int RS = a.RS;
    float* Qt = (float*)(bp + L.qoff);
    for (int bx = lane; bx * kBoxCols < ncopy; bx += 32)
        tma_q_box(Qt + (size_t)bx * kBoxCols * RS, qmap, mt.a0, bx * kBoxCols, bar);
    if (lane == 31 && j >= 1) bulk_g2s(bp + L.roff, a.rt + mt.a0, cbytes, bar);
    if (lane == 30) bulk_g2s(bp + L.foff, a.f0 + mt.a0, cbytes, bar);
    if (D > 1 && lane == 29) bulk_g2s(bp + L.foff + sizeof(float) * RS, a.f1 + mt.a0, cbytes, bar);
    if (D > 2 && lane == 28) bulk_g2s(bp + L.foff + 2 * sizeof(float) * RS, a.f2 + mt.a0, cbytes, bar);
    if (lane == 27) bulk_g2s(bp + L.ioff, a.item_start + mt.ia0, ibytes, bar);
    if (lane == 26) bulk_g2s(bp + L.coff, a.item_cell + mt.ia0, ibytes, bar);
    if (D <= 2 && mt.zspan > 0 && lane == 25) bulk_g2s(bp, a.z + mt.zlo, (unsigned)mt.zspan * 8u, bar);
}

// The one-read pass F_j.  Persistent CTAs walk the tiles with a two-stage TMA pipeline:
// while tile t is processed from shared memory, the bulk copies of the next tile are in flight.
template <int D, int CMAX, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) fused_pass_kernel(FusedArgs a, const __grid_constant__ CUtensorMap qmap) {
    using A = typename AccT<float, D>::type;
    constexpr int S = Slots<D>::value;
    extern __shared__ __align__(128) unsigned char smraw[];
    const LanczosState& st = a.st;
    const int j = *st.jdev;
    if (st.flags[0]) return;
    const int k = a.k, RS = a.RS;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int nw = NT / 32;
    const BufLayout L = buf_layout(k, RS, a.IS, D);
    // ---- shared memory carve-up
    uint64_t* bars = (uint64_t*)smraw;
    TileMeta* tinfo = (TileMeta*)(smraw + 16);
    unsigned char* sp = smraw + 128;
    unsigned char* buf0 = sp;                       sp += 2 * L.stride;     // 128-B aligned
    double* part = (double*)sp;                     sp += sizeof(double) * 2 * (k + 1);
    float* rnew = (float*)sp;                       sp += sizeof(float) * RS;
    float* wts = (float*)sp;                        // [D][4][RS] (also the update's partials)
    sp += sizeof(float) * (4 * D * RS > 2048 ? 4 * D * RS : 2048);
    int* litem = (int*)sp;                          sp += sizeof(int) * RS;
    float* csf = (float*)sp;
    // ---- per-step scalars
    double s1 = 0.0, a1 = 0.0, b2 = 0.0;
    if (j >= 1) {
        s1 = st.qscale[j - 1];
        a1 = st.alpha[j - 1] * s1;
        b2 = j >= 2 ? st.beta[j - 2] * st.qscale[j - 2] : 0.0;
    }
    for (int i = tid; i < j; i += NT) csf[i] = (float)st.cvec[i];
    const A sig = (A)a.sigma2;
    const int ncols = j + 1;
    const bool moments = j < k - 1;
    float ga[CMAX], gb[CMAX];               // per-lane Gram partials of columns wid + nw*c
#pragma unroll
    for (int c = 0; c < CMAX; ++c) ga[c] = gb[c] = 0.f;
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (wid == 0)
        for (int bb = 0; bb < 2; ++bb) {
            const int64_t t = blockIdx.x + (int64_t)bb * gridDim.x;
            if (t < a.n_tiles)
                issue_tile<D>(a, &qmap, j, load_meta(a.meta, t), &tinfo[bb], &bars[bb], buf0 + bb * L.stride, L);
        }
    unsigned phases = 0u;                   // bit b = parity of buffer b's next phase
    int b = 0;
    for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x, b ^= 1) {
        // descriptor of the tile this buffer takes next, fetched early so that its latency
        // hides behind this tile's work
        const int64_t tn = t + 2 * (int64_t)gridDim.x;
        TileMeta next{};
        if (wid == 0 && tn < a.n_tiles) next = load_meta(a.meta, tn);
        mbar_wait(&bars[b], (phases >> b) & 1u);
        phases ^= 1u << b;
        const TileMeta ti = tinfo[b];
        if (a.debug_mode == 1) {            // experiment: TMA streaming only
            __syncthreads();
            if (wid == 0 && tn < a.n_tiles) issue_tile<D>(a, &qmap, j, next, &tinfo[b], &bars[b], buf0 + b * L.stride, L);
            continue;
        }
        unsigned char* bp = buf0 + b * L.stride;
        float* Qt = (float*)(bp + L.qoff);
        const float* rprev = (const float*)(bp + L.roff);
        const float* fr = (const float*)(bp + L.foff);
        const int* ist = (const int*)(bp + L.ioff);        // item_start[ia0 ...]
        const int* icl = (const int*)(bp + L.coff);        // item_cell[ia0 ...]
        const double* zs = (const double*)bp;
        const int it0 = ti.it0, it1 = ti.it1, p0 = ti.p0, a0 = ti.a0, nch = ti.nch, ia0 = ti.ia0;
        const int off = p0 - a0, rows = ti.p1 - p0;
        float* qj = Qt + (size_t)j * RS;
        // ---- lagged three-term + CGS update of column j.  Thread (cg, rq) sums the columns
        //      i = cg, cg + NCG, ... of the correction for the 4 aligned rows of quad rq; the
        //      NCG partial sums meet in shared memory.  Rows outside the tile are written as 0
        //      so later phases work on whole 16-byte chunks.  The upper half of the block maps
        //      rows to (tile-local) items meanwhile.
        constexpr int NCG = NT / 64;
        float4* red = reinterpret_cast<float4*>(wts);      // [NCG][64] partials (wts is free here)
        if (j >= 1) {
            const int rq = tid & 63, cg = tid >> 6;
            if (rq < nch) {
                float4 cr = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int i = cg; i < j; i += NCG) {
                    const float ci = csf[i];
                    const float4 v = *reinterpret_cast<const float4*>(Qt + (size_t)i * RS + rq * 4);
                    cr.x += ci * v.x; cr.y += ci * v.y; cr.z += ci * v.z; cr.w += ci * v.w;
                }
                red[cg * 64 + rq] = cr;
            }
        }
        if (tid >= NT / 2) {
            for (int it = it0 + tid - NT / 2; it < it1; it += NT / 2) {
                const int q1 = ist[it + 1 - ia0] - a0;
                for (int rr = ist[it - ia0] - a0; rr < q1; ++rr) litem[rr] = it - ia0;
            }
        }
        __syncthreads();
        if (j >= 1 && tid < nch) {
            const int r0 = tid * 4;
            float4 cr = red[tid];
#pragma unroll
            for (int g2 = 1; g2 < NCG; ++g2) {
                const float4 v = red[g2 * 64 + tid];
                cr.x += v.x; cr.y += v.y; cr.z += v.z; cr.w += v.w;
            }
            const float4 rp4 = *reinterpret_cast<const float4*>(rprev + r0);
            const float4 q1 = *reinterpret_cast<const float4*>(Qt + (size_t)(j - 1) * RS + r0);
            float4 q2 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (j >= 2) q2 = *reinterpret_cast<const float4*>(Qt + (size_t)(j - 2) * RS + r0);
            const float rps[4] = {rp4.x, rp4.y, rp4.z, rp4.w}, q1s[4] = {q1.x, q1.y, q1.z, q1.w};
            const float q2s[4] = {q2.x, q2.y, q2.z, q2.w}, crs[4] = {cr.x, cr.y, cr.z, cr.w};
            float out[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int rr = r0 + e;
                const bool in = rr >= off && rr < off + rows;
                const double rp = s1 * (double)rps[e] - a1 * (double)q1s[e] - b2 * (double)q2s[e];
                out[e] = in ? (float)(rp - (double)crs[e]) : 0.f;
                if (in) a.Q[(int64_t)j * a.ldq + a0 + rr] = out[e];
            }
            *reinterpret_cast<float4*>(qj + r0) = make_float4(out[0], out[1], out[2], out[3]);
        }
        __syncthreads();
        // ---- Keys weights of every row (kept for the moments) and the gather
        //      r~_j = W^T z~_j + sigma^2 Q~_j (0 outside the tile)
        for (int rr = tid; rr < 4 * nch; rr += NT) {
            const bool in = rr >= off && rr < off + rows;
            float rv = 0.f;
            if (in) {
                A w0[4], w1[4], w2[4];
                keys4<A>((A)fr[rr], w0);
                if (D > 1) keys4<A>((A)fr[RS + rr], w1);
                if (D > 2) keys4<A>((A)fr[2 * RS + rr], w2);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    wts[e * RS + rr] = (float)w0[e];
                    if (D > 1) wts[(4 + e) * RS + rr] = (float)w1[e];
                    if (D > 2) wts[(8 + e) * RS + rr] = (float)w2[e];
                }
                A zl[S];
                const int base = stencil_base<D>(a.g, icl[litem[rr]]);
                if (D <= 2 && ti.zspan > 0) load_stencil<A, D>(a.g, zs - ti.zlo, base, zl);
                else load_stencil<A, D>(a.g, a.z, base, zl);
                rv = (float)(stencil_dot<A, D>(w0, w1, w2, zl) + sig * (A)qj[rr]);
            } else if (j == 0) {
                qj[rr] = 0.f;           // the probe column was staged with its neighbours' rows
            }
            rnew[rr] = rv;
        }
        __syncthreads();
        // ---- stencil moments of r~_j (M) and of Q~_j (M2 = exact W Q~_j): one (slot, item)
        //      unit per thread over the item's rows, weights from shared memory
        if (moments) {
            const int nit = it1 - it0;
            for (int e = tid; e < S * nit; e += NT) {
                const int l = e / nit, li = it0 - ia0 + (e - l * nit);
                const int la = D == 1 ? l : (D == 2 ? l >> 2 : l >> 4);
                const int lb = D == 2 ? (l & 3) : ((l >> 2) & 3);
                const int lc = l & 3;
                const int q0 = ist[li] - a0, q1 = ist[li + 1] - a0;
                A accr = A(0), accq = A(0);
                for (int rr = q0; rr < q1; ++rr) {
                    float w = wts[la * RS + rr];
                    if (D > 1) w *= wts[(4 + lb) * RS + rr];
                    if (D > 2) w *= wts[(8 + lc) * RS + rr];
                    accr += (A)w * (A)rnew[rr];
                    accq += (A)w * (A)qj[rr];
                }
                a.M[(int64_t)l * a.n_items + ia0 + li] = (double)accr;
                a.M2[(int64_t)l * a.n_items + ia0 + li] = (double)accq;
            }
        }
        for (int tt = tid; tt < rows; tt += NT) a.rt[p0 + tt] = rnew[off + tt];
        // ---- Gram sums (warps own columns, lanes own 16-byte chunks, partials stay in lanes)
        float4 rn4[3], qj4[3];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int ch = lane + 32 * u;
            const bool ok = ch < nch;
            rn4[u] = ok ? *reinterpret_cast<const float4*>(rnew + ch * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
            qj4[u] = ok ? *reinterpret_cast<const float4*>(qj + ch * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int c = 0; c < CMAX; ++c) {
            const int col = wid + nw * c;
            if (col < ncols) {
                const float* qc = Qt + (size_t)col * RS;
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int ch = lane + 32 * u;
                    if (ch < nch) {
                        const float4 v = *reinterpret_cast<const float4*>(qc + ch * 4);
                        ga[c] += v.x * rn4[u].x + v.y * rn4[u].y + v.z * rn4[u].z + v.w * rn4[u].w;
                        gb[c] += v.x * qj4[u].x + v.y * qj4[u].y + v.z * qj4[u].z + v.w * qj4[u].w;
                    }
                }
            }
        }
        __syncthreads();        // buffer b, rnew, wts and litem are free again
        if (wid == 0 && tn < a.n_tiles) issue_tile<D>(a, &qmap, j, next, &tinfo[b], &bars[b], bp, L);
    }
#pragma unroll
    for (int c = 0; c < CMAX; ++c) {
        const int col = wid + nw * c;
        const double da = warp_sum((double)ga[c]), db = warp_sum((double)gb[c]);
        if (lane == 0 && col < ncols) {
            part[col] = da;
            part[k + 1 + col] = db;
        }
    }
    __syncthreads();
    double* AB = st.AB + (int64_t)j * 2 * (k + 1);
    for (int i = tid; i < ncols; i += NT) {
        atomicAdd(&AB[i], part[i]);
        atomicAdd(&AB[k + 1 + i], part[k + 1 + i]);
    }
}

// ---- scalars of step j (one CTA): beta_{j-1}, s_j, alpha_j, row j of the Cholesky of T,
// breakdown (reading A12), then the next pass's reorthogonalisation coefficients
//   c_{j,i} = q_i^T r'_j = s_i s_j A_i - alpha_j s_i s_j B_i - beta_{j-1} s_i s_{j-1} G_{i,j-1}
// with G_{i,j-1} = Q~_i . Q~_{j-1} (previous pass' B, or this pass' B_{j-1} for i = j).
__global__ void fused_scalars_kernel(LanczosState st, int k, double tol) {
    const int j = *st.jdev;
    int* fl = st.flags;
    if (fl[0]) return;
    __shared__ double sh[4];
    __shared__ int stop;
    const double* Aj = st.AB + (int64_t)j * 2 * (k + 1);
    const double* Bj = Aj + (k + 1);
    if (threadIdx.x == 0) {
        stop = 0;
        const double Bjj = Bj[j];
        double sj = 0.0, bjm1 = 0.0;
        if (j == 0) {
            if (!(Bjj > 0.0)) {
                fl[3] = 1; fl[0] = 1; fl[1] = 0; stop = 1;
            } else {
                st.bnorm2[0] = Bjj;
                sj = 1.0 / sqrt(Bjj);
            }
        } else {
            bjm1 = sqrt(Bjj);
            const double bmax = fmax(st.amax_bmax[1], bjm1);
            st.amax_bmax[1] = bmax;
            if (!(bjm1 >= tol * (st.amax_bmax[0] + 2.0 * bmax))) {
                fl[0] = 1; fl[1] = j; stop = 1;
            } else {
                st.beta[j - 1] = bjm1;
                st.Ls[j - 1] = bjm1 / st.Ld[j - 1];
                sj = 1.0 / bjm1;
            }
        }
        if (!stop) {
            st.qscale[j] = sj;
            const double aj = sj * sj * Aj[j];
            st.alpha[j] = aj;
            st.amax_bmax[0] = fmax(st.amax_bmax[0], fabs(aj));
            const double lsub = j > 0 ? st.Ls[j - 1] : 0.0;
            const double piv = aj - lsub * lsub;
            if (!(piv > 0.0)) {
                fl[2] = 1; fl[0] = 1; fl[1] = j; stop = 1;
            } else {
                const double ld = sqrt(piv);
                st.Ld[j] = ld;
                st.g[j] = (j == 0) ? 1.0 / ld : -lsub * st.g[j - 1] / ld;
                if (j == k - 1) { fl[0] = 1; fl[1] = k; stop = 1; }
            }
            sh[0] = sj; sh[1] = aj; sh[2] = bjm1; sh[3] = j > 0 ? st.qscale[j - 1] : 0.0;
        }
    }
    __syncthreads();
    if (stop) return;
    const double sj = sh[0], aj = sh[1], bjm1 = sh[2], sjm1 = sh[3];
    const double* Bprev = j > 0 ? st.AB + (int64_t)(j - 1) * 2 * (k + 1) + (k + 1) : nullptr;
    for (int i = threadIdx.x; i <= j; i += blockDim.x) {
        const double si = i == j ? sj : st.qscale[i];
        const double G = j == 0 ? 0.0 : (i <= j - 1 ? Bprev[i] : Bj[j - 1]);
        const double c = si * sj * Aj[i] - aj * si * sj * Bj[i] - bjm1 * si * sjm1 * G;
        const double cs = c * si;
        st.cvec[i] = cs;
        double gm = cs;
        if (i == j) gm += aj * sj;
        if (i == j - 1) gm += bjm1 * sjm1;
        st.gam[i] = gm;
    }
}

// ---- m side of step j, one thread per grid node:
//   Rc[:, j] = (s_j z~_j - L_{j,j-1} Rc[:, j-1]) / L_jj ;  a += ||b|| g_j Rc[:, j]
//   wr = (W r~_j)[i], wq = (W Q~_j)[i] from the moments of pass F_j
//   (mode 1: write wr, wq to wbuf and stop, for the all-reduce; mode 2: read them back)
//   u~_j := wq (the exact scatter of the stored column replaces the recurrence value, so
//   rounding errors are not propagated through the three-term recurrence of the u~), then
//   u~_{j+1} = s_j wr - sum_i gamma_i u~_i  -> U64[(j+1)%3], U32[j+1], u
template <int D>
__global__ void __launch_bounds__(256) fused_mside_kernel(GridDev g, LanczosState st, int k, int64_t n_items,
                                                          const int* __restrict__ cis, const double* __restrict__ M,
                                                          const double* __restrict__ M2,
                                                          const double* __restrict__ z, double* __restrict__ Rc,
                                                          double* __restrict__ amean, int mean_y,
                                                          double* __restrict__ U64, float* __restrict__ U32,
                                                          double* __restrict__ u, double* __restrict__ wbuf,
                                                          int mode) {
    __shared__ float gs[1024];
    const int j = *st.jdev;
    const int* fl = st.flags;
    const int m = g.m_total;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = !fl[0] && j < k - 1;
    if (active && mode != 1)
        for (int t = threadIdx.x; t < j - 1 && t < 1024; t += blockDim.x) gs[t] = (float)st.gam[t];
    __syncthreads();
    if (i >= m) return;
    if (mode != 2 && j < fl[1] && !fl[2] && !fl[3]) {
        const double prev = j > 0 ? Rc[(int64_t)(j - 1) * m + i] : 0.0;
        const double v = (st.qscale[j] * z[i] - (j > 0 ? st.Ls[j - 1] : 0.0) * prev) / st.Ld[j];
        Rc[(int64_t)j * m + i] = v;
        if (mean_y) amean[i] += sqrt(st.bnorm2[0]) * st.g[j] * v;
    }
    if (!active) return;
    double wr, wq;
    if (mode == 2) {
        wr = wbuf[i];
        wq = wbuf[m + i];
    } else {
        wr = node_pull<D>(g, n_items, cis, M, i);
        wq = node_pull<D>(g, n_items, cis, M2, i);
        if (mode == 1) {
            wbuf[i] = wr;
            wbuf[m + i] = wq;
            return;
        }
    }
    U64[(int64_t)(j % 3) * m + i] = wq;
    U32[(int64_t)j * m + i] = (float)wq;
    double un = st.qscale[j] * wr - st.gam[j] * wq;
    if (j >= 1) un -= st.gam[j - 1] * U64[(int64_t)((j - 1) % 3) * m + i];
    float corr = 0.f;
    for (int t = 0; t < j - 1; ++t) corr += (t < 1024 ? gs[t] : (float)st.gam[t]) * U32[(int64_t)t * m + i];
    un -= (double)corr;
    U64[(int64_t)((j + 1) % 3) * m + i] = un;
    U32[(int64_t)(j + 1) * m + i] = (float)un;
    u[i] = un;
}

__global__ void fused_init_u_kernel(const double* __restrict__ u0, double* __restrict__ U64, float* __restrict__ U32,
                                    int m) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        U64[i] = u0[i];
        U32[i] = (float)u0[i];
    }
}

__global__ void advance_kernel(int* jdev) {
    if (threadIdx.x == 0) jdev[0] += 1;
}

// tile t = items whose first point lies in [t*Rp, (t+1)*Rp); items have <= kItemMax points
__global__ void tile_setup_kernel(const int* __restrict__ item_start, int64_t n_items, int Rp, int64_t n_tiles,
                                  int* __restrict__ tile_first) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_tiles;
         t += (int64_t)gridDim.x * blockDim.x)
        tile_first[t] = (int)n_items;
}
__global__ void tile_assign_kernel(const int* __restrict__ item_start, int64_t n_items, int Rp, int64_t n_tiles,
                                   int* __restrict__ tile_first) {
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t hi = item_start[it] / Rp;
        const int64_t lo = it == 0 ? 0 : item_start[it - 1] / Rp + 1;
        for (int64_t t = lo; t <= hi && t < n_tiles; ++t) tile_first[t] = (int)it;
    }
}

__global__ void tile_meta_kernel(const int* __restrict__ tile_first, const int* __restrict__ item_start,
                                 const int* __restrict__ item_cell, int64_t n_tiles, GridDev g,
                                 TileMeta* __restrict__ meta) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        TileMeta mt;
        mt.it0 = tile_first[t];
        mt.it1 = tile_first[t + 1];
        mt.p0 = item_start[mt.it0];
        mt.p1 = item_start[mt.it1];
        mt.a0 = mt.p0 & ~3;
        mt.nch = (mt.p1 - mt.a0 + 3) >> 2;
        mt.ia0 = mt.it0 & ~3;
        mt.nich = (mt.it1 + 1 - mt.ia0 + 3) >> 2;
        mt.zlo = 0;
        mt.zspan = 0;
        if (g.d <= 2 && mt.it1 > mt.it0) {
            const int cmin = item_cell[mt.it0], cmax = item_cell[mt.it1 - 1];
            const int lo = g.d == 1 ? cmin - 1 : cmin - g.stride[0] - 1;
            const int hi = g.d == 1 ? cmax + 2 : cmax + 2 * g.stride[0] + 2;
            mt.zlo = lo & ~1;
            const int span = (hi - mt.zlo + 2) & ~1;
            mt.zspan = span <= kZMax ? span : 0;
        }
        mt.pad0 = mt.pad1 = 0;
        meta[t] = mt;
    }
}

void launch_fused_pass(Cache& c, cudaStream_t s) {
    FusedArgs a;
    a.g = c.g;
    a.ldq = c.ldq;
    a.n_items = c.n_items;
    a.n_tiles = c.n_tiles;
    a.k = c.k_req;
    a.RS = c.tile_cap + 8;
    a.IS = c.tile_cap + 16;
    a.Q = (float*)c.Q;
    a.rt = (float*)c.r;
    a.f0 = (const float*)c.frac[0];
    a.f1 = (const float*)c.frac[1];
    a.f2 = (const float*)c.frac[2];
    a.item_cell = c.item_cell;
    a.item_start = c.item_start;
    a.meta = (const TileMeta*)c.tile_meta;
    a.z = (const double*)c.z[0];
    a.sigma2 = c.sigma2;
    a.M = (double*)c.M;
    a.M2 = (double*)c.M2;
    a.st = c.st;
    a.debug_mode = std::getenv("LOVE_FUSED_DEBUG") ? std::atoi(std::getenv("LOVE_FUSED_DEBUG")) : 0;
    const size_t sm = fused_smem(a.k, a.RS, a.IS, c.g.d);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device);
    const int NT = c.fused_threads;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(c.n_tiles, (int64_t)nsm * (512 / NT)));
    const int cneed = (int)ceil_div(a.k + 1, NT / 32);
#define LOVE_FUSED(DD, CM, NTT)                                                        \
    do {                                                                               \
        ensure_smem((const void*)fused_pass_kernel<DD, CM, NTT>, sm);                  \
        LOVE_LAUNCH((fused_pass_kernel<DD, CM, NTT>), grid, NTT, sm, s, a, *(const CUtensorMap*)c.qmap); \
    } while (0)
#define LOVE_FUSED_NT(DD, CM)                              \
    do {                                                   \
        if (NT == 256) LOVE_FUSED(DD, CM, 256);            \
        else LOVE_FUSED(DD, CM, 512);                      \
    } while (0)
#define LOVE_FUSED_D(DD)                          \
    do {                                          \
        if (cneed <= 4) LOVE_FUSED_NT(DD, 4);     \
        else if (cneed <= 8) LOVE_FUSED_NT(DD, 8); \
        else LOVE_FUSED_NT(DD, 16);               \
    } while (0)
    switch (c.g.d) {
        case 1: LOVE_FUSED_D(1); break;
        case 2: LOVE_FUSED_D(2); break;
        default: LOVE_FUSED_D(3); break;
    }
#undef LOVE_FUSED_D
#undef LOVE_FUSED_NT
#undef LOVE_FUSED
}

void launch_mside(Cache& c, int mode, double* wbuf, cudaStream_t s) {
    const int gm = (int)ceil_div(c.g.m_total, 256);
#define LOVE_MSIDE(DD)                                                                                          \
    LOVE_LAUNCH(fused_mside_kernel<DD>, gm, 256, 0, s, c.g, c.st, c.k_req, c.n_items, c.cell_item_start,        \
                (const double*)c.M, (const double*)c.M2, (const double*)c.z[0], (double*)c.Rc_col, (double*)c.a, \
                c.probe == LOVE_PROBE_Y ? 1 : 0, c.U64, c.U32, (double*)c.u, wbuf, mode)
    switch (c.g.d) {
        case 1: LOVE_MSIDE(1); break;
        case 2: LOVE_MSIDE(2); break;
        default: LOVE_MSIDE(3); break;
    }
#undef LOVE_MSIDE
}

// one Lanczos step (the index lives in device memory); j_host only addresses the
// multi-GPU all-reduces of eager mode
void enqueue_fused_step(Cache& c, int j_host, double* wbuf, cudaStream_t s) {
    const int k = c.k_req;
    const int m = c.g.m_total;
    {
        ProfScope ps(LOVE_PROF_FUSED_PASS, s);
        launch_fused_pass(c, s);
    }
    if (c.comm != nullptr) {
        ProfScope ps(LOVE_PROF_COMM, s);
        allreduce_sum(c, c.st.AB + (int64_t)j_host * 2 * (k + 1), 2 * (k + 1), true, s);
    }
    {
        ProfScope ps(LOVE_PROF_SCALARS, s);
        LOVE_LAUNCH(fused_scalars_kernel, 1, 256, 0, s, c.st, k, c.tol);
    }
    {
        ProfScope ps(LOVE_PROF_SCATTER, s);
        if (c.comm != nullptr) {
            launch_mside(c, 1, wbuf, s);
            {
                ProfScope pc(LOVE_PROF_COMM, s);
                allreduce_sum(c, wbuf, 2 * (int64_t)m, true, s);
            }
            launch_mside(c, 2, wbuf, s);
        } else {
            launch_mside(c, 0, wbuf, s);
        }
    }
    {
        ProfScope ps(LOVE_PROF_KUU, s);
        launch_kuu(c, (const double*)c.u, (double*)c.z[0], s);
    }
    LOVE_LAUNCH(advance_kernel, 1, 32, 0, s, c.st.jdev);
}

}  // namespace

// tiles, U buffers; called by the build before the Lanczos loop (fp32 mode)
void setup_fused(Cache& c, cudaStream_t s) {
    const int k = c.k_req;
    // 512 threads, one CTA per SM with 192-row tiles, or 256 threads, two CTAs per SM with
    // smaller tiles (LOVE_FUSED_NT overrides; both double-buffer their tiles)
    int NT = 512;
    if (const char* e = std::getenv("LOVE_FUSED_NT")) NT = std::atoi(e) == 256 ? 256 : 512;
    const size_t budget = NT == 512 ? 220 * 1024 : 110 * 1024;
    int cap = NT == 512 ? 192 : 128;
    while (cap > 64 && fused_smem(k, cap + 8, cap + 16, c.g.d) > budget) cap -= 32;
    if (fused_smem(k, cap + 8, cap + 16, c.g.d) > budget || k + 1 > 16 * (NT / 32) || cap - kItemMax < kItemMax) {
        c.fused = false;             // very large k: classical mode
        return;
    }
    c.fused_threads = NT;
    c.tile_cap = cap;
    {   // tensor map of Q~ (column-major, ldq x (k+1) fp32) with {RS rows, 8 columns} boxes
        using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        static EncodeFn encode = nullptr;
        if (!encode) {
            cudaDriverEntryPointQueryResult q;
            void* fn = nullptr;
            cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
                       "cuTensorMapEncodeTiled lookup");
            if (q != cudaDriverEntryPointSuccess || !fn) throw LoveError{LOVE_ERR_CUDA, "cuTensorMapEncodeTiled missing"};
            encode = (EncodeFn)fn;
        }
        const cuuint64_t dims[2] = {(cuuint64_t)c.ldq, (cuuint64_t)(k + 1)};
        const cuuint64_t strides[1] = {(cuuint64_t)c.ldq * sizeof(float)};
        const cuuint32_t box[2] = {(cuuint32_t)(cap + 8), (cuuint32_t)kBoxCols};
        const cuuint32_t estr[2] = {1, 1};
        CUtensorMap* m = (CUtensorMap*)c.qmap;
        const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c.Q, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw LoveError{LOVE_ERR_CUDA, "cuTensorMapEncodeTiled failed"};
    }
    const int Rp = cap - kItemMax;
    c.n_tiles = ceil_div(c.n, Rp);
    c.tile_first = (int*)dalloc(c, sizeof(int) * (c.n_tiles + 1), s);
    LOVE_LAUNCH(tile_setup_kernel, (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(c.n_tiles + 1, 256), 1024)),
                256, 0, s, c.item_start, c.n_items, Rp, c.n_tiles, c.tile_first);
    if (c.n_items > 0)
        LOVE_LAUNCH(tile_assign_kernel, (int)std::min<int64_t>(ceil_div(c.n_items, 256), 4096), 256, 0, s,
                    c.item_start, c.n_items, Rp, c.n_tiles, c.tile_first);
    c.tile_meta = dalloc(c, sizeof(TileMeta) * std::max<int64_t>(c.n_tiles, 1), s);
    if (c.n_tiles > 0)
        LOVE_LAUNCH(tile_meta_kernel, (int)std::min<int64_t>(ceil_div(c.n_tiles, 256), 4096), 256, 0, s,
                    c.tile_first, c.item_start, c.item_cell, c.n_tiles, c.g, (TileMeta*)c.tile_meta);
    const int m = c.g.m_total;
    c.U64 = (double*)dalloc(c, sizeof(double) * 3 * (size_t)m, s);
    c.U32 = (float*)dalloc(c, sizeof(float) * (size_t)(k + 1) * m, s);
    const size_t K = k;
    c.st.AB = (double*)dalloc(c, sizeof(double) * K * 2 * (K + 1), s);
    c.M2 = dalloc(c, sizeof(double) * (size_t)(1 << (2 * c.g.d)) * std::max<int64_t>(c.n_items, 1), s);
    c.st.cvec = (double*)dalloc(c, sizeof(double) * (K + 1), s);
    c.st.gam = (double*)dalloc(c, sizeof(double) * (K + 1), s);
}

void run_lanczos_fused(Cache& c, cudaStream_t s) {
    const int k = c.k_req;
    const int m = c.g.m_total;
    double* wbuf = nullptr;
    if (c.comm != nullptr) cuda_check(cudaMallocAsync((void**)&wbuf, sizeof(double) * 2 * (size_t)m, s), "wbuf alloc");
    {   // u~_0 = W Q~_0 (the probe b) and z~_0 = K_UU u~_0
        ProfScope ps(LOVE_PROF_SCATTER, s);
        const StepRef ref{nullptr, 0, c.one, nullptr};
        launch_scatter<float>(c, (const float*)c.Q, ref, (double*)c.u, s);
        if (c.comm != nullptr) {
            ProfScope pc(LOVE_PROF_COMM, s);
            allreduce_sum(c, c.u, m, true, s);
        }
        LOVE_LAUNCH(fused_init_u_kernel, (int)std::min<int64_t>(ceil_div(m, 256), 2048), 256, 0, s,
                    (const double*)c.u, c.U64, c.U32, m);
    }
    {
        ProfScope ps(LOVE_PROF_KUU, s);
        launch_kuu(c, (const double*)c.u, (double*)c.z[0], s);
    }
    const bool graph = c.comm == nullptr && !profiling() && std::getenv("LOVE_NO_GRAPH") == nullptr;
    if (graph) {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        const int64_t before = g_launch_count.load();      // captured launches run once per replay
        cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
        enqueue_fused_step(c, 0, wbuf, s);
        cuda_check(cudaStreamEndCapture(s, &g), "end capture");
        cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
        const int64_t nodes = g_launch_count.load() - before;
        g_launch_count -= nodes;
        for (int j = 0; j < k; ++j) {
            cuda_check(cudaGraphLaunch(ge, s), "graph launch");
            g_launch_count += nodes;
        }
        cuda_check(cudaGraphExecDestroy(ge), "graph destroy");
        cuda_check(cudaGraphDestroy(g), "graph destroy");
    } else {
        for (int j = 0; j < k; ++j) enqueue_fused_step(c, j, wbuf, s);
    }
    if (wbuf) cuda_check(cudaFreeAsync(wbuf, s), "wbuf free");
}

}  // namespace love
