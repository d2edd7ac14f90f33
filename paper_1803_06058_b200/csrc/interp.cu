// interp.cu -- interpolation index/weight builder and the one-time cell sort.
//
// SKI cubic interpolation: each point x is expressed by the 4 closest grid nodes
// per dimension (Keys cubic, reading A2), 4^d nonzeros in w_x.  We store per point only its
// cell (fp64 floor, reading A3) and the fractional offset per dimension; the 4^d weights are
// recomputed on the fly in every kernel (8d -> 4d bytes per point per pass in fp32 mode).
// Points are counting-sorted by flat cell once per build and cut into work items of at most
// kItemMax consecutive points of one cell: every later pass streams them in that order.
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

#include "love_internal.h"

namespace love {

namespace {

__global__ void interp_points_kernel(GridDev g, const double* __restrict__ X, int64_t n,
                                     int* __restrict__ cell, double* __restrict__ frac64,
                                     int* __restrict__ range_flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int flat = 0;
        bool bad = false;
        for (int d = 0; d < g.d; ++d) {
            const double s = (X[i * g.d + d] - g.lo[d]) / g.h[d];
            const double jf = floor(s);
            const double f = s - jf;
            // stencil j-1..j+2 must lie in [0, m-1] (reading A4); NaN fails both tests
            bad |= !(jf >= 1.0 && jf <= (double)(g.m[d] - 3));
            const int j = bad ? 1 : (int)jf;
            flat += j * g.stride[d];
            frac64[i * g.d + d] = bad ? 0.0 : f;
        }
        cell[i] = bad ? 0 : flat;
        if (bad) atomicOr(range_flag, 1);
    }
}

__global__ void histogram_kernel(const int* __restrict__ cell, int64_t n, int* __restrict__ count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&count[cell[i]], 1);
}

// ---- three-phase exclusive scan of int32 (out has L+1 entries, out[L] = total)
constexpr int kScanThreads = 1024, kScanPer = 4, kScanChunk = kScanThreads * kScanPer;

__device__ int block_exclusive_scan(int v, int* sm) {   // sm: 32 ints
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = (lane < (int)(blockDim.x >> 5)) ? sm[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sm[lane] = s;
    }
    __syncthreads();
    const int base = wid > 0 ? sm[wid - 1] : 0;
    __syncthreads();
    return base + x - v;
}

__global__ void scan_reduce_kernel(const int* __restrict__ in, int64_t L, int* __restrict__ bsum) {
    __shared__ int sm[32];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    int v = 0;
    for (int e = 0; e < kScanPer; ++e) {
        const int64_t i = base + (int64_t)threadIdx.x * kScanPer + e;
        if (i < L) v += in[i];
    }
    v = block_sum(v, sm);
    if (threadIdx.x == 0) bsum[blockIdx.x] = v;
}

__global__ void scan_blocksums_kernel(int* __restrict__ bsum, int nb) {
    __shared__ int sm[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int s = 0; s < nb; s += blockDim.x) {
        const int i = s + threadIdx.x;
        const int v = i < nb ? bsum[i] : 0;
        const int ex = block_exclusive_scan(v, sm);
        const int c0 = carry;
        if (i < nb) bsum[i] = c0 + ex;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = c0 + ex + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[nb] = carry;
}

__global__ void scan_apply_kernel(const int* __restrict__ in, int64_t L, const int* __restrict__ bsum,
                                  int* __restrict__ out) {
    __shared__ int sm[32];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    int v[kScanPer];
    int tot = 0;
    for (int e = 0; e < kScanPer; ++e) {
        const int64_t i = base + (int64_t)threadIdx.x * kScanPer + e;
        v[e] = i < L ? in[i] : 0;
        tot += v[e];
    }
    int ex = block_exclusive_scan(tot, sm) + bsum[blockIdx.x];
    for (int e = 0; e < kScanPer; ++e) {
        const int64_t i = base + (int64_t)threadIdx.x * kScanPer + e;
        if (i < L) out[i] = ex;
        ex += v[e];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[L] = bsum[gridDim.x];
}

void exclusive_scan(const int* in, int64_t L, int* out, cudaStream_t s) {
    const int nb = (int)ceil_div(L, kScanChunk);
    int* bsum = nullptr;
    cuda_check(cudaMallocAsync((void**)&bsum, sizeof(int) * (nb + 1), s), "scan alloc");
    LOVE_LAUNCH(scan_reduce_kernel, nb, kScanThreads, 0, s, in, L, bsum);
    LOVE_LAUNCH(scan_blocksums_kernel, 1, kScanThreads, 0, s, bsum, nb);
    LOVE_LAUNCH(scan_apply_kernel, nb, kScanThreads, 0, s, in, L, bsum, out);
    cuda_check(cudaFreeAsync(bsum, s), "scan free");
}

__global__ void place_kernel(const int* __restrict__ cell, int64_t n, const int* __restrict__ start,
                             int* __restrict__ fill, int* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = cell[i];
        perm[start[c] + atomicAdd(&fill[c], 1)] = (int)i;
    }
}

// Deterministic order inside a cell (by original index): insertion sort per cell.  Cells
// larger than 4096 points keep the atomic order (only the summation order changes).
__global__ void sort_within_cells_kernel(const int* __restrict__ start, int m_total,
                                         int* __restrict__ perm) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m_total) return;
    const int b = start[c], e = start[c + 1];
    if (e - b < 2 || e - b > 4096) return;
    for (int i = b + 1; i < e; ++i) {
        const int v = perm[i];
        int j = i - 1;
        while (j >= b && perm[j] > v) {
            perm[j + 1] = perm[j];
            --j;
        }
        perm[j + 1] = v;
    }
}

// The same order (ascending original index within each cell) by rank instead of insertion:
// a group of 8 lanes per cell, every entry's rank = the count of smaller entries of its cell
// (entries are distinct point indices), written to out.  O(n^2 / 8) per cell against the
// insertion sort's dependent O(n^2) global moves on one thread (cfg4's densest cells hold ~330
// points); 8-lane groups keep the grid small for the many empty and few-point cells.
constexpr int kRankLanes = 8;
__global__ void rank_within_cells_kernel(const int* __restrict__ start, int m_total, const int* __restrict__ perm,
                                         int* __restrict__ out) {
    const int sub = threadIdx.x & (kRankLanes - 1);
    const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kRankLanes;
    if (c >= m_total) return;                         // whole groups leave together
    const int b = start[c], e = start[c + 1], n = e - b;
    if (n > 4096) {                                   // as the insertion sort: left in place order
        for (int i = sub; i < n; i += kRankLanes) out[b + i] = perm[b + i];
        return;
    }
    for (int i = sub; i < n; i += kRankLanes) {
        const int v = perm[b + i];
        int rank = 0;
        for (int j = 0; j < n; ++j) rank += perm[b + j] < v;
        out[b + rank] = v;
    }
}

template <typename V>
__global__ void gather_sorted_kernel(int d, const int* __restrict__ perm, int64_t n,
                                     const double* __restrict__ frac64, const double* __restrict__ y,
                                     V* __restrict__ f0, V* __restrict__ f1, V* __restrict__ f2,
                                     V* __restrict__ b, const int* __restrict__ cell, int* __restrict__ pcell) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int o = perm[p];
        if (pcell != nullptr) pcell[p] = cell[o];
        f0[p] = (V)frac64[(int64_t)o * d + 0];
        if (d > 1) f1[p] = (V)frac64[(int64_t)o * d + 1];
        if (d > 2) f2[p] = (V)frac64[(int64_t)o * d + 2];
        b[p] = (V)y[o];
    }
}

__global__ void items_per_cell_kernel(const int* __restrict__ start, int m_total, int* __restrict__ nit, int imax) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m_total) return;
    nit[c] = (int)ceil_div(start[c + 1] - start[c], imax);
}

__global__ void build_items_kernel(const int* __restrict__ start, const int* __restrict__ item0,
                                   int m_total, int64_t n, int* __restrict__ item_cell,
                                   int* __restrict__ item_start, int imax) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m_total) return;
    const int b = start[c], e = start[c + 1];
    const int it0 = item0[c];
    // ceil(cnt / kItemMax) items of (nearly) equal size: the lanes of a warp loop alike
    const int cnt = e - b, nit = (cnt + imax - 1) / imax;
    for (int i = 0; i < nit; ++i) {
        item_cell[it0 + i] = c;
        item_start[it0 + i] = b + (int)((int64_t)i * cnt / nit);
    }
    if (c == m_total - 1) item_start[item0[m_total]] = (int)n;
}

// points per item: kItemMax (LOVE_ITEM_MAX = 1 .. kItemMax: measurement switch)
inline int item_max() {
    static const int v = std::getenv("LOVE_ITEM_MAX") ? std::atoi(std::getenv("LOVE_ITEM_MAX")) : kItemMax;
    return v >= 1 && v <= kItemMax ? v : kItemMax;
}

inline int grid_for(int64_t n, int threads) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 148 * 32));
}

}  // namespace

void counting_sort_keys(const int* keys, int64_t n, int nbins, int* start, int* perm, cudaStream_t s) {
    int* count = nullptr;
    cuda_check(cudaMallocAsync((void**)&count, sizeof(int) * (nbins + 1), s), "sort alloc");
    cuda_check(cudaMemsetAsync(count, 0, sizeof(int) * (nbins + 1), s), "sort memset");
    if (n > 0) LOVE_LAUNCH(histogram_kernel, grid_for(n, 256), 256, 0, s, keys, n, count);
    exclusive_scan(count, nbins, start, s);
    cuda_check(cudaMemsetAsync(count, 0, sizeof(int) * (nbins + 1), s), "sort memset");
    if (n > 0) LOVE_LAUNCH(place_kernel, grid_for(n, 256), 256, 0, s, keys, n, start, count, perm);
    cuda_check(cudaFreeAsync(count, s), "sort free");
}

void launch_interp_points(const Cache& c, const double* X, int64_t n, int* cell, double* frac64,
                          int* range_flag, cudaStream_t s) {
    if (n == 0) return;
    LOVE_LAUNCH(interp_points_kernel, grid_for(n, 256), 256, 0, s, c.g, X, n, cell, frac64,
                range_flag);
}

void launch_counting_sort(Cache& c, const int* cell, const double* frac64, const double* y,
                          int64_t n, void* b_out, cudaStream_t s) {
    const int M = c.g.m_total;
    int* count = nullptr;
    cuda_check(cudaMallocAsync((void**)&count, sizeof(int) * (M + 1), s), "sort alloc");
    cuda_check(cudaMemsetAsync(count, 0, sizeof(int) * (M + 1), s), "sort memset");
    if (n > 0) LOVE_LAUNCH(histogram_kernel, grid_for(n, 256), 256, 0, s, cell, n, count);
    exclusive_scan(count, M, c.cell_start, s);
    cuda_check(cudaMemsetAsync(count, 0, sizeof(int) * (M + 1), s), "sort memset");
    if (n > 0) {
        LOVE_LAUNCH(place_kernel, grid_for(n, 256), 256, 0, s, cell, n, c.cell_start, count, c.perm);
        if (std::getenv("LOVE_INSERTION_SORT") != nullptr) {
            LOVE_LAUNCH(sort_within_cells_kernel, (int)ceil_div(M, 128), 128, 0, s, c.cell_start, M, c.perm);
        } else {
            int* ranked = nullptr;
            cuda_check(cudaMallocAsync((void**)&ranked, sizeof(int) * n, s), "rank alloc");
            LOVE_LAUNCH(rank_within_cells_kernel, (int)ceil_div((int64_t)M * kRankLanes, 256), 256, 0, s, c.cell_start,
                        M, c.perm, ranked);
            cuda_check(cudaMemcpyAsync(c.perm, ranked, sizeof(int) * n, cudaMemcpyDeviceToDevice, s), "rank copy");
            cuda_check(cudaFreeAsync(ranked, s), "rank free");
        }
        if (c.precision == LOVE_FP64)
            LOVE_LAUNCH(gather_sorted_kernel<double>, grid_for(n, 256), 256, 0, s, c.g.d, c.perm, n,
                        frac64, y, (double*)c.frac[0], (double*)c.frac[1], (double*)c.frac[2],
                        (double*)b_out, cell, c.pcell);
        else
            LOVE_LAUNCH(gather_sorted_kernel<float>, grid_for(n, 256), 256, 0, s, c.g.d, c.perm, n,
                        frac64, y, (float*)c.frac[0], (float*)c.frac[1], (float*)c.frac[2],
                        (float*)b_out, cell, c.pcell);
    }
    LOVE_LAUNCH(items_per_cell_kernel, (int)ceil_div(M, 256), 256, 0, s, c.cell_start, M, count, item_max());
    exclusive_scan(count, M, c.cell_item_start, s);
    cuda_check(cudaFreeAsync(count, s), "sort free");
}

int64_t count_items_host(Cache& c, cudaStream_t s) {
    int nit = 0;
    cuda_check(cudaMemcpyAsync(&nit, c.cell_item_start + c.g.m_total, sizeof(int),
                               cudaMemcpyDeviceToHost, s), "items d2h");
    cuda_check(cudaStreamSynchronize(s), "items sync");
    return nit;
}

void launch_build_items(Cache& c, cudaStream_t s) {
    const int M = c.g.m_total;
    LOVE_LAUNCH(build_items_kernel, (int)ceil_div(M, 256), 256, 0, s, c.cell_start,
                c.cell_item_start, M, c.n, c.item_cell, c.item_start, item_max());
}

}  // namespace love
