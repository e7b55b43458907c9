// fph_mask.cu -- candidate masks: per simplex, the cloud points inside its
// masking ball, as ascending cloud indices.
//
// Replaces reference floodph/filtration.py:130 compute_mask (one axis slab
// per batch, then per simplex the slab points with |x - c|^2 <= 2 r r, c and
// r the Ritter ball of floodph/geometry.py:123).  Here the ball is answered
// from the device grid (fph_grid.cu, built with the point permutation):
// every grid row of the ball's cell box is one contiguous run of sorted
// points, each tested with the reference's float64 expression
// sq64(x, c) <= (2 r) r.  One warp per simplex: a count pass, a scan, a fill
// pass, then a segmented sort restores ascending cloud indices.  The
// reference's fallbacks for an EMPTY ball (the batch slab, then the whole
// cloud) depend on batch composition and stay with the host caller.
#include <cub/cub.cuh>

#include "fph_dev.cuh"
#include "fph_grid.cuh"

namespace fph {

namespace {

struct MaskBall {
    double c[3];
    double r2;   // (2 r) r, the reference's closed-ball bound on |x - c|^2
    double rad;  // query radius for the cell box: sqrt(2) r with slack
};

__device__ __forceinline__ MaskBall mask_ball(const double* lm3, const int* cells, int s, int k) {
    Verts V;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int id = j <= k ? cells[(size_t)s * 4 + j] : -1;
        V.v[j][0] = id >= 0 ? lm3[(size_t)id * 3 + 0] : 0.0;
        V.v[j][1] = id >= 0 ? lm3[(size_t)id * 3 + 1] : 0.0;
        V.v[j][2] = id >= 0 ? lm3[(size_t)id * 3 + 2] : 0.0;
    }
    MaskBall b;
    const double r = ritter(V, k, b.c);
    b.r2 = __dmul_rn(__dmul_rn(2.0, r), r);
    b.rad = 1.4142135623730951 * r * (1.0 + 1e-9) + 1e-300;
    return b;
}

// kFill = false: out_count[s] = number of cloud points in the ball of s;
// kFill = true: their cloud indices (unordered) at out_idx[offsets[s] ...]
template <bool kFill>
__global__ void mask_kernel(const Grid* __restrict__ gp, const double* __restrict__ lm3,
                            const int* __restrict__ cells, int n, int k, long long* __restrict__ out_count,
                            const long long* __restrict__ offsets, int* __restrict__ out_idx) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const Grid g = *gp;
    const MaskBall b = mask_ball(lm3, cells, warp, k);
    const Box box = ball_box(g, b.c[0], b.c[1], b.c[2], b.rad);
    const int rows = box.rows();
    long long cnt = 0;
    long long pos = kFill ? offsets[warp] : 0;
    for (int r = 0; r < rows; ++r) {
        const int2 run = row_run(g, box, r, b.c[0], b.c[1], b.c[2], b.rad, true);
        for (int i0 = run.x; i0 < run.y; i0 += 32) {
            const int i = i0 + lane;
            const bool in = i < run.y && sq64(g.x[i], g.y[i], g.z[i], b.c[0], b.c[1], b.c[2]) <= b.r2;
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            if (kFill && in) out_idx[pos + __popc(bal & ((1u << lane) - 1u))] = g.idx[i];
            pos += __popc(bal);
            cnt += __popc(bal);
        }
    }
    if (!kFill && lane == 0) out_count[warp] = cnt;
}

}  // namespace

int candidate_counts(const Grid* g, const double* d_lm3, const int* d_cells4, int n, int k,
                     long long* d_counts, cudaStream_t stream) {
    if (n == 0) return FPH_OK;
    mask_kernel<false><<<(unsigned)(((long long)n * 32 + 255) / 256), 256, 0, stream>>>(
        g, d_lm3, d_cells4, n, k, d_counts, nullptr, nullptr);
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

int candidate_fill(const Grid* g, const double* d_lm3, const int* d_cells4, int n, int k,
                   const long long* d_offsets, long long total, int* d_idx,
                   cudaStream_t stream) {
    if (n == 0 || total == 0) return FPH_OK;
    mask_kernel<true><<<(unsigned)(((long long)n * 32 + 255) / 256), 256, 0, stream>>>(
        g, d_lm3, d_cells4, n, k, nullptr, d_offsets, d_idx);
    FPH_CUDA_TRY(cudaGetLastError());
    // ascending cloud indices per simplex (the reference sorts its slab)
    Scratch sc(stream);
    int* sorted = nullptr;
    FPH_TRY(sc.alloc(&sorted, (size_t)total));
    size_t tmp_bytes = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, d_idx, sorted, total, n, d_offsets,
                                       d_offsets + 1, stream);
    unsigned char* tmp = nullptr;
    FPH_TRY(sc.alloc(&tmp, tmp_bytes));
    FPH_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, d_idx, sorted, total, n,
                                                    d_offsets, d_offsets + 1, stream));
    FPH_CUDA_TRY(cudaMemcpyAsync(d_idx, sorted, sizeof(int) * total, cudaMemcpyDeviceToDevice,
                                 stream));
    return FPH_OK;
}

}  // namespace fph
