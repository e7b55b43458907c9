// fph_grid.cu -- GPU-built uniform spatial grid over the cloud.
//
// The reference restricts each simplex's minimisation to the cloud points in
// its sqrt(2)-inflated Ritter ball, found through an axis-sorted slab
// (floodph/filtration.py:130 compute_mask, floodph/spatial.py:22).  Here the
// cloud is binned once into a uniform grid: points are radix-sorted by
// linear cell id (x fastest) and stored as float64 SoA, so every (y, z) row
// of a ball's cell box is ONE contiguous run of points -- coalesced loads and
// a two-lookup range query per row.  cell_start is the exclusive scan of the
// per-cell histogram; the points are placed by a stable radix sort of their
// cell ids and a gather (see gather_kernel).
#include <cub/cub.cuh>

#include <cmath>
#include <algorithm>
#include <cstdio>

#include "fph_grid.cuh"

namespace fph {

namespace {

__device__ __forceinline__ unsigned long long d2ord(double d) {
    unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double ord2d(unsigned long long u) {
    unsigned long long v = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
    double d;
    memcpy(&d, &v, sizeof(d));
    return d;
}

// bbox[0..2] = ordered mins, bbox[3..5] = ordered maxes.  The cloud is read
// as one flat array of n * dim doubles, consecutive threads on consecutive
// elements (fully coalesced; row-wise reads of the 24-byte rows ran at a
// third of HBM speed); the grid stride is a multiple of dim, so a thread
// always sees the same axis.  Block reduction per axis, then one atomic per
// block and value.
constexpr int kBoxThreads = 384;  // a multiple of 2 and 3

__global__ void __launch_bounds__(kBoxThreads) bbox_kernel(const double* __restrict__ pts, int n,
                                                           int dim, unsigned long long* bbox) {
    __shared__ double smn[3][kBoxThreads / 32], smx[3][kBoxThreads / 32];
    const long long total = (long long)n * dim;
    const long long stride = (long long)gridDim.x * kBoxThreads;
    const long long e0 = (long long)blockIdx.x * kBoxThreads + threadIdx.x;
    const int axis = (int)(e0 % dim);
    double mn = INFINITY, mx = -INFINITY;
    long long e = e0;
    for (; e + 3 * stride < total; e += 4 * stride) {  // four loads in flight
        const double v0 = pts[e], v1 = pts[e + stride], v2 = pts[e + 2 * stride],
                     v3 = pts[e + 3 * stride];
        mn = fmin(mn, fmin(fmin(v0, v1), fmin(v2, v3)));
        mx = fmax(mx, fmax(fmax(v0, v1), fmax(v2, v3)));
    }
    for (; e < total; e += stride) {
        mn = fmin(mn, pts[e]);
        mx = fmax(mx, pts[e]);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int a = 0; a < dim; ++a) {
        double lo = axis == a ? mn : INFINITY, hi = axis == a ? mx : -INFINITY;
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (l == 0) {
            smn[a][w] = lo;
            smx[a][w] = hi;
        }
    }
    __syncthreads();
    if (threadIdx.x < dim) {
        const int a = threadIdx.x;
        double lo = smn[a][0], hi = smx[a][0];
        for (int i = 1; i < kBoxThreads / 32; ++i) {
            lo = fmin(lo, smn[a][i]);
            hi = fmax(hi, smx[a][i]);
        }
        atomicMin(&bbox[a], d2ord(lo));
        atomicMax(&bbox[3 + a], d2ord(hi));
    }
}

// Grid parameters from the box, on the device (one thread): cell edge
// h = (volume x occupancy / n)^(1/dim) (each extent clamped below at 1e-3 of
// the largest), grown by 1.25x until the cell count fits the host-allocated
// capacity.  The host never reads the box back, so nothing waits for it.
__global__ void grid_params_kernel(const unsigned long long* __restrict__ bbox, int n, int dim,
                                   double cell_size, double occupancy, long long cap,
                                   Grid out, Grid* __restrict__ g) {
    double lo[3] = {0.0, 0.0, 0.0}, hi[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < dim; ++a) {
        lo[a] = ord2d(bbox[a]);
        hi[a] = ord2d(bbox[3 + a]);
    }
    double h = cell_size;
    if (!(h > 0.0)) {
        double emax = 0.0;
        for (int a = 0; a < dim; ++a) emax = fmax(emax, hi[a] - lo[a]);
        if (!(emax > 0.0)) {
            h = 1.0;
        } else {
            double vol = 1.0;
            for (int a = 0; a < dim; ++a) vol *= fmax(hi[a] - lo[a], emax * 1e-3);
            h = pow(vol * occupancy / (double)n, 1.0 / dim);
            if (!(h > 0.0)) h = emax;
        }
    }
    int nc[3] = {1, 1, 1};
    for (int attempt = 0; attempt < 256; ++attempt) {
        double total = 1.0;
        for (int a = 0; a < dim; ++a) {
            const double c = floor((hi[a] - lo[a]) / h) + 1.0;
            nc[a] = (int)fmin(c, (double)(1 << 24));
            total *= nc[a];
        }
        if (total <= (double)cap) break;
        h *= 1.25;
    }
    out.n = n;  // `out` arrives with the host-set fields (the pointers)
    out.nx = nc[0];
    out.ny = nc[1];
    out.nz = dim == 3 ? nc[2] : 1;
    out.lox = lo[0];
    out.loy = lo[1];
    out.loz = dim == 3 ? lo[2] : 0.0;
    out.h = h;
    out.inv_h = 1.0 / h;
    double scale = 0.0;
    for (int a = 0; a < dim; ++a) scale = fmax(scale, fmax(fabs(lo[a]), fabs(hi[a])));
    out.margin = 1e-9 * (scale + h);
    *g = out;
}

// cell id per point + histogram (counting sort pass 1)
__global__ void cell_id_kernel(const double* __restrict__ pts, int n, int dim,
                               const Grid* __restrict__ gp, int* __restrict__ keys,
                               int* __restrict__ counts) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Grid g = *gp;
    const double* p = pts + (size_t)i * dim;
    int ix = cell_coord(p[0], g.lox, g.inv_h, g.nx);
    int iy = cell_coord(p[1], g.loy, g.inv_h, g.ny);
    int iz = dim == 3 ? cell_coord(p[2], g.loz, g.inv_h, g.nz) : 0;
    const int key = (iz * g.ny + iy) * g.nx + ix;
    keys[i] = key;
    atomicAdd(counts + key, 1);
}

// counting sort pass 3: each point to its cell's next free slot.  The order
// inside a cell is arbitrary -- nothing downstream depends on it (minima are
// order-free, the float64 refine is exact).
__global__ void scatter_kernel(const double* __restrict__ pts, int n, int dim,
                               const int* __restrict__ keys, const int* __restrict__ cell_start,
                               int* __restrict__ cursor, double* __restrict__ x,
                               double* __restrict__ y, double* __restrict__ z,
                               int* __restrict__ idx) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int key = keys[i];
    const int pos = cell_start[key] + atomicAdd(cursor + key, 1);
    const double* p = pts + (size_t)i * dim;
    x[pos] = p[0];
    y[pos] = p[1];
    z[pos] = dim == 3 ? p[2] : 0.0;
    if (idx) idx[pos] = i;
}

// points in cell order: sorted position i takes the point sorted_idx[i]
// (a gather -- coalesced writes, one 24-byte random read per point -- where
// an atomic-cursor scatter made 3 random 8-byte writes per point: 1.29 ms
// vs a few hundred microseconds at 10M points).  A stable radix sort keeps
// the points of a cell in cloud order, so the layout is deterministic.
__global__ void gather_kernel(const double* __restrict__ pts, int n, int dim,
                              const int* __restrict__ sorted_idx, double* __restrict__ x,
                              double* __restrict__ y, double* __restrict__ z,
                              int* __restrict__ idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int j = sorted_idx[i];
    const double* p = pts + (size_t)j * dim;
    x[i] = p[0];
    y[i] = p[1];
    z[i] = dim == 3 ? p[2] : 0.0;
    if (idx) idx[i] = j;
}

__global__ void iota_kernel(int* __restrict__ out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

}  // namespace

int grid_build(const double* d_pts, int n, int dim, double cell_size, double occupancy,
               cudaStream_t stream, GridStore* gs, bool keep_index) {
    if (n < 1 || (dim != 2 && dim != 3)) {
        set_error("grid_build: need n >= 1 and dim in {2, 3}");
        return FPH_EARG;
    }
    gs->free_all(stream);
    // cell capacity: about n / occupancy cells for a cloud filling its box;
    // rounding adds at most ~30% for realistic shapes, and the device grows h
    // until the grid fits (coarser cells stay exact, only slower)
    const long long cap = std::min<long long>(
        1ll << 27, (long long)(2.0 * n / (occupancy > 0 ? occupancy : 2.0)) + 4096);
    Scratch sc(stream);
    unsigned long long* d_bbox = nullptr;
    // clouds that fit L2 scatter with an atomic cursor per cell; larger ones
    // sort (cell id, index) and gather (random writes to a 240 MB array cost
    // 1.29 ms at 10M points, the sort + gather 0.5 ms; below 2M points the
    // sort's fixed cost loses)
    const bool sorted_path = n > (1 << 21);
    int *keys = nullptr, *counts = nullptr, *cursor = nullptr;
    FPH_TRY(sc.alloc(&d_bbox, 6));
    FPH_TRY(sc.alloc(&keys, n));
    FPH_TRY(sc.alloc(&counts, cap + 1));
    if (!sorted_path) {
        FPH_TRY(sc.alloc(&cursor, cap));
        FPH_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(int) * cap, stream));
    }
    // +2: a 16-byte aligned bulk copy of a run may read one point past the end
    FPH_CUDA_TRY(cudaMallocAsync(&gs->x, sizeof(double) * (n + 2), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->y, sizeof(double) * (n + 2), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->z, sizeof(double) * (n + 2), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->cell_start, sizeof(int) * (cap + 1), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->d_grid, sizeof(Grid), stream));
    if (keep_index) FPH_CUDA_TRY(cudaMallocAsync(&gs->idx, sizeof(int) * n, stream));
    Grid g{};
    g.x = gs->x;
    g.y = gs->y;
    g.z = gs->z;
    g.cell_start = gs->cell_start;
    g.idx = gs->idx;
    FPH_CUDA_TRY(cudaMemsetAsync(d_bbox, 0xff, 3 * sizeof(unsigned long long), stream));
    FPH_CUDA_TRY(cudaMemsetAsync(d_bbox + 3, 0, 3 * sizeof(unsigned long long), stream));
    FPH_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int) * (cap + 1), stream));
    const long long elems = (long long)n * dim;
    const int blocks = (int)std::min<long long>(4 * 148, (elems + 4 * kBoxThreads - 1) / (4 * kBoxThreads));
    bbox_kernel<<<blocks, kBoxThreads, 0, stream>>>(d_pts, n, dim, d_bbox);
    grid_params_kernel<<<1, 1, 0, stream>>>(d_bbox, n, dim, cell_size, occupancy, cap, g,
                                            gs->d_grid);
    cell_id_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_pts, n, dim, gs->d_grid, keys, counts);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, gs->cell_start, (int)(cap + 1),
                                  stream);
    unsigned char* tmp = nullptr;
    FPH_TRY(sc.alloc(&tmp, tmp_bytes));
    FPH_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, gs->cell_start,
                                               (int)(cap + 1), stream));
    if (!sorted_path) {
        scatter_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_pts, n, dim, keys, gs->cell_start,
                                                            cursor, gs->x, gs->y, gs->z, gs->idx);
        FPH_CUDA_TRY(cudaGetLastError());
        gs->cap = cap;
        return FPH_OK;
    }
    int *keys_sorted = nullptr, *iota = nullptr, *order = nullptr;
    FPH_TRY(sc.alloc(&keys_sorted, n));
    FPH_TRY(sc.alloc(&iota, n));
    FPH_TRY(sc.alloc(&order, n));
    iota_kernel<<<(n + 255) / 256, 256, 0, stream>>>(iota, n);
    int end_bit = 1;
    while ((1ll << end_bit) < cap) ++end_bit;
    size_t sort_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys, keys_sorted, iota, order, n, 0,
                                    end_bit, stream);
    unsigned char* sort_tmp = nullptr;
    FPH_TRY(sc.alloc(&sort_tmp, sort_bytes));
    FPH_CUDA_TRY(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, keys, keys_sorted, iota,
                                                 order, n, 0, end_bit, stream));
    gather_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_pts, n, dim, order, gs->x, gs->y, gs->z,
                                                       gs->idx);
    FPH_CUDA_TRY(cudaGetLastError());
    gs->cap = cap;
    return FPH_OK;
}

void GridStore::free_all(cudaStream_t stream) {
    for (void* p : {(void*)x, (void*)y, (void*)z, (void*)cell_start, (void*)idx, (void*)d_grid})
        if (p) cudaFreeAsync(p, stream);
    x = y = z = nullptr;
    cell_start = nullptr;
    idx = nullptr;
    d_grid = nullptr;
}

}  // namespace fph
