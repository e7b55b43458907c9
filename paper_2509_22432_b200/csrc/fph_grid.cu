// fph_grid.cu -- GPU-built uniform spatial grid over the cloud.
//
// The reference restricts each simplex's minimisation to the cloud points in
// its sqrt(2)-inflated Ritter ball, found through an axis-sorted slab
// (floodph/filtration.py:130 compute_mask, floodph/spatial.py:22).  Here the
// cloud is binned once into a uniform grid: points are radix-sorted by
// linear cell id (x fastest) and stored as float64 SoA, so every (y, z) row
// of a ball's cell box is ONE contiguous run of points -- coalesced loads and
// a two-lookup range query per row.  Binning is a counting sort (histogram,
// scan, scatter): cell_start is the scan itself.
#include <cub/cub.cuh>

#include <cmath>
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

// bbox[0..2] = ordered mins, bbox[3..5] = ordered maxes (block reduction,
// then one atomic per block and value)
__global__ void bbox_kernel(const double* __restrict__ pts, int n, int dim,
                            unsigned long long* bbox) {
    __shared__ double smn[3][32], smx[3][32];
    double mn[3] = {INFINITY, INFINITY, INFINITY};
    double mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        for (int a = 0; a < dim; ++a) {
            double v = pts[(size_t)i * dim + a];
            mn[a] = fmin(mn[a], v);
            mx[a] = fmax(mx[a], v);
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int a = 0; a < dim; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmax(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
        if (l == 0) {
            smn[a][w] = mn[a];
            smx[a][w] = mx[a];
        }
    }
    __syncthreads();
    if (threadIdx.x < dim) {
        const int a = threadIdx.x;
        double lo = smn[a][0], hi = smx[a][0];
        for (int i = 1; i < nw; ++i) {
            lo = fmin(lo, smn[a][i]);
            hi = fmax(hi, smx[a][i]);
        }
        atomicMin(&bbox[a], d2ord(lo));
        atomicMax(&bbox[3 + a], d2ord(hi));
    }
}

// cell id per point + histogram (counting sort pass 1)
__global__ void cell_id_kernel(const double* __restrict__ pts, int n, int dim, Grid g,
                               int* __restrict__ keys, int* __restrict__ counts) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
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

}  // namespace

double grid_cell_size(const double lo[3], const double hi[3], int dim, long long n,
                      double occupancy) {
    double ext[3];
    double emax = 0.0;
    for (int a = 0; a < dim; ++a) {
        ext[a] = hi[a] - lo[a];
        emax = fmax(emax, ext[a]);
    }
    if (!(emax > 0.0)) return 1.0;
    double vol = 1.0;
    for (int a = 0; a < dim; ++a) vol *= fmax(ext[a], emax * 1e-3);
    double h = pow(vol * occupancy / (double)(n > 0 ? n : 1), 1.0 / dim);
    return h > 0.0 ? h : emax;
}

int grid_build(const double* d_pts, int n, int dim, double cell_size, double occupancy,
               cudaStream_t stream, GridStore* gs, bool keep_index) {
    if (n < 1 || (dim != 2 && dim != 3)) {
        set_error("grid_build: need n >= 1 and dim in {2, 3}");
        return FPH_EARG;
    }
    unsigned long long hb[6];
    unsigned long long* d_bbox = nullptr;
    FPH_CUDA_TRY(cudaMallocAsync(&d_bbox, 6 * sizeof(unsigned long long), stream));
    // ordered-int identities: mins start at ~0, maxes at 0 (no host copy)
    FPH_CUDA_TRY(cudaMemsetAsync(d_bbox, 0xff, 3 * sizeof(unsigned long long), stream));
    FPH_CUDA_TRY(cudaMemsetAsync(d_bbox + 3, 0, 3 * sizeof(unsigned long long), stream));
    int blocks = (n + 255) / 256;
    if (blocks > 592) blocks = 592;
    bbox_kernel<<<blocks, 256, 0, stream>>>(d_pts, n, dim, d_bbox);
    FPH_CUDA_TRY(cudaMemcpyAsync(hb, d_bbox, sizeof(hb), cudaMemcpyDeviceToHost, stream));
    FPH_CUDA_TRY(cudaStreamSynchronize(stream));
    FPH_CUDA_TRY(cudaFreeAsync(d_bbox, stream));
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) {
        lo[a] = ord2d(hb[a]);
        hi[a] = ord2d(hb[3 + a]);
    }
    double h = cell_size > 0.0 ? cell_size : grid_cell_size(lo, hi, dim, n, occupancy);
    const double max_cells = 1 << 27;
    int nc[3] = {1, 1, 1};
    for (int attempt = 0; attempt < 64; ++attempt) {
        double total = 1.0;
        for (int a = 0; a < dim; ++a) {
            double c = floor((hi[a] - lo[a]) / h) + 1.0;
            nc[a] = (int)fmin(c, 1 << 24);
            total *= nc[a];
        }
        if (total <= max_cells) break;
        h *= 1.25;
    }
    Grid g{};
    g.n = n;
    g.nx = nc[0];
    g.ny = nc[1];
    g.nz = dim == 3 ? nc[2] : 1;
    g.lox = lo[0];
    g.loy = lo[1];
    g.loz = dim == 3 ? lo[2] : 0.0;
    g.h = h;
    g.inv_h = 1.0 / h;
    double scale = 0.0;
    for (int a = 0; a < dim; ++a) scale = fmax(scale, fmax(fabs(lo[a]), fabs(hi[a])));
    g.margin = 1e-9 * (scale + h);
    long long ncells = (long long)g.nx * g.ny * g.nz;

    gs->free_all(stream);
    int *keys = nullptr, *counts = nullptr, *cursor = nullptr;
    FPH_CUDA_TRY(cudaMallocAsync(&keys, sizeof(int) * n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int) * (ncells + 1), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&cursor, sizeof(int) * ncells, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->x, sizeof(double) * n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->y, sizeof(double) * n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->z, sizeof(double) * n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&gs->cell_start, sizeof(int) * (ncells + 1), stream));
    if (keep_index) FPH_CUDA_TRY(cudaMallocAsync(&gs->idx, sizeof(int) * n, stream));
    FPH_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int) * (ncells + 1), stream));
    FPH_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(int) * ncells, stream));
    cell_id_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_pts, n, dim, g, keys, counts);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, gs->cell_start, ncells + 1, stream);
    void* tmp = nullptr;
    FPH_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, stream));
    FPH_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, gs->cell_start, ncells + 1,
                                               stream));
    scatter_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_pts, n, dim, keys, gs->cell_start, cursor,
                                                        gs->x, gs->y, gs->z, gs->idx);
    FPH_CUDA_TRY(cudaGetLastError());
    FPH_CUDA_TRY(cudaFreeAsync(tmp, stream));
    FPH_CUDA_TRY(cudaFreeAsync(keys, stream));
    FPH_CUDA_TRY(cudaFreeAsync(counts, stream));
    FPH_CUDA_TRY(cudaFreeAsync(cursor, stream));
    g.x = gs->x;
    g.y = gs->y;
    g.z = gs->z;
    g.cell_start = gs->cell_start;
    g.idx = gs->idx;
    gs->grid = g;
    gs->ncells = ncells;
    return FPH_OK;
}

void GridStore::free_all(cudaStream_t stream) {
    if (x) cudaFreeAsync(x, stream);
    if (y) cudaFreeAsync(y, stream);
    if (z) cudaFreeAsync(z, stream);
    if (cell_start) cudaFreeAsync(cell_start, stream);
    if (idx) cudaFreeAsync(idx, stream);
    x = y = z = nullptr;
    cell_start = nullptr;
    idx = nullptr;
}

}  // namespace fph
