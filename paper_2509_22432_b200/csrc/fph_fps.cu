// fph_fps.cu -- farthest point sampling as one persistent cooperative kernel.
//
// Replaces reference floodph/geometry.py:88 farthest_point_sampling
// (numpy loop: d2 = |X - X[start]|^2, d2[start] = -1; repeat: nxt =
// argmax(d2) (first maximiser), d2 = minimum(d2, |X - X[nxt]|^2),
// d2[nxt] = -1).  Bit-exact: the squared distances use the reference's
// float64 accumulation order (sq64) and the argmax keeps the lowest index
// among equal values, so the landmark sequence is identical.
//
// Layout: one CTA per SM (cooperative launch, all CTAs co-resident), each
// owning a contiguous slice of the cloud.  When a slice fits, its float64
// coordinates live in shared memory (SoA) and the running minimum in
// registers for the whole run -- a 1M-point cloud never touches HBM after
// the first load.  Larger clouds stream coordinates and the running minimum
// through L2/HBM.  Per iteration each CTA publishes its (value, index) to a
// double-buffered slot array and bumps one monotone arrival counter; one
// thread per CTA polls the counter (ld.acquire) until all CTAs of this
// iteration arrived, then the CTA reads every slot in one coalesced pass.
// All CTAs reduce the same slots in the same order, so they agree on the
// next landmark without a second broadcast.
#include "fph_common.cuh"

namespace fph {

namespace {

constexpr int kFpsThreads = 1024;
constexpr int kFpsMaxPT = 9;  // points per thread in the shared-memory variant

struct __align__(16) Slot {
    double val;
    int idx;
    int pad;
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void better(double& bv, int& bi, double v, int i) {
    if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
    }
}

__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int oi = __shfl_xor_sync(0xffffffffu, i, o);
        better(v, i, ov, oi);
    }
}

// Block-wide argmax; result valid in every thread.
__device__ __forceinline__ void block_argmax(double& v, int& i, double* sv, int* si) {
    warp_argmax(v, i);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) {
        sv[w] = v;
        si[w] = i;
    }
    __syncthreads();
    int nw = blockDim.x >> 5;
    if (w == 0) {
        v = l < nw ? sv[l] : -INFINITY;
        i = l < nw ? si[l] : 0x7fffffff;
        warp_argmax(v, i);
        if (l == 0) {
            sv[0] = v;
            si[0] = i;
        }
    }
    __syncthreads();
    v = sv[0];
    i = si[0];
}

template <bool kSmem>
__global__ void __launch_bounds__(kFpsThreads, 1)
    fps_kernel(const double* __restrict__ px, const double* __restrict__ py,
               const double* __restrict__ pz, int n, int k, int start, int chunk,
               double* __restrict__ mind, Slot* slots, unsigned long long* arrived,
               long long* __restrict__ out) {
    extern __shared__ double sm[];
    __shared__ double red_v[32];
    __shared__ int red_i[32];
    const int G = gridDim.x;
    const int beg = blockIdx.x * chunk;
    const int end = min(n, beg + chunk);
    const int cnt = max(0, end - beg);
    double* sx = sm;
    double* sy = sm + chunk;
    double* sz = sm + 2 * chunk;
    double md[kSmem ? kFpsMaxPT : 1];
    if (kSmem) {
        for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
            sx[j] = px[beg + j];
            sy[j] = py[beg + j];
            sz[j] = pz[beg + j];
        }
#pragma unroll
        for (int t = 0; t < kFpsMaxPT; ++t) md[t] = INFINITY;
        __syncthreads();
    } else {
        for (int j = threadIdx.x; j < cnt; j += blockDim.x) mind[beg + j] = INFINITY;
    }
    int cur = start;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = start;
    for (int it = 1; it <= k; ++it) {
        const double qx = px[cur], qy = py[cur], qz = pz[cur];
        double bv = -INFINITY;
        int bi = 0x7fffffff;
        if (kSmem) {
#pragma unroll
            for (int t = 0; t < kFpsMaxPT; ++t) {
                int j = threadIdx.x + t * kFpsThreads;
                if (j < cnt) {
                    int gi = beg + j;
                    double d = sq64(sx[j], sy[j], sz[j], qx, qy, qz);
                    double m = gi == cur ? -1.0 : fmin(md[t], d);
                    md[t] = m;
                    better(bv, bi, m, gi);
                }
            }
        } else {
            for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
                int gi = beg + j;
                double d = sq64(px[gi], py[gi], pz[gi], qx, qy, qz);
                double m = gi == cur ? -1.0 : fmin(mind[gi], d);
                mind[gi] = m;
                better(bv, bi, m, gi);
            }
        }
        if (it == k) break;
        block_argmax(bv, bi, red_v, red_i);
        Slot* buf = slots + (it & 1) * G;
        if (threadIdx.x == 0) {
            buf[blockIdx.x].val = bv;
            buf[blockIdx.x].idx = bi;
            __threadfence();
            atomicAdd(arrived, 1ull);
            const unsigned long long target = (unsigned long long)G * it;
            while (ld_acquire(arrived) < target) {
            }
        }
        __syncthreads();
        // every CTA has published this iteration's candidate
        double v = -INFINITY;
        int i = 0x7fffffff;
        for (int b = threadIdx.x; b < G; b += blockDim.x) {
            double sv = __ldcg(&buf[b].val);
            int si = __ldcg(&buf[b].idx);
            better(v, i, sv, si);
        }
        block_argmax(v, i, red_v, red_i);
        cur = i;
        if (blockIdx.x == 0 && threadIdx.x == 0) out[it] = cur;
    }
}

}  // namespace

int fps_run(const double* d_x, const double* d_y, const double* d_z, int n, int k, int start,
            long long* d_out, cudaStream_t stream) {
    if (k < 1 || k > n || start < 0 || start >= n) {
        set_error("farthest point sampling: need 1 <= k <= n and 0 <= start < n");
        return FPH_EARG;
    }
    int dev = 0;
    FPH_CUDA_TRY(cudaGetDevice(&dev));
    int sms = 0;
    FPH_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int max_smem = 0;
    FPH_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    int G = sms;
    int chunk = (n + G - 1) / G;
    size_t smem = (size_t)chunk * 3 * sizeof(double);
    bool use_smem = chunk <= kFpsThreads * kFpsMaxPT && smem + 1024 <= (size_t)max_smem;
    if (n < 4096) {
        G = (n + 1023) / 1024;  // tiny clouds: few CTAs, less barrier traffic
        chunk = (n + G - 1) / G;
        smem = (size_t)chunk * 3 * sizeof(double);
        use_smem = true;
    }
    Slot* slots = nullptr;
    double* mind = nullptr;
    unsigned long long* arrived = nullptr;
    FPH_CUDA_TRY(cudaMallocAsync(&slots, sizeof(Slot) * 2 * G, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&arrived, sizeof(unsigned long long), stream));
    FPH_CUDA_TRY(cudaMemsetAsync(arrived, 0, sizeof(unsigned long long), stream));
    if (!use_smem) FPH_CUDA_TRY(cudaMallocAsync(&mind, sizeof(double) * n, stream));
    void* args[] = {(void*)&d_x,   (void*)&d_y,  (void*)&d_z,   (void*)&n,
                    (void*)&k,     (void*)&start, (void*)&chunk, (void*)&mind,
                    (void*)&slots, (void*)&arrived, (void*)&d_out};
    if (use_smem) {
        FPH_CUDA_TRY(cudaFuncSetAttribute(fps_kernel<true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        FPH_CUDA_TRY(cudaLaunchCooperativeKernel((void*)fps_kernel<true>, dim3(G),
                                                 dim3(kFpsThreads), args, smem, stream));
    } else {
        FPH_CUDA_TRY(cudaLaunchCooperativeKernel((void*)fps_kernel<false>, dim3(G),
                                                 dim3(kFpsThreads), args, 0, stream));
    }
    FPH_CUDA_TRY(cudaGetLastError());
    FPH_CUDA_TRY(cudaFreeAsync(slots, stream));
    FPH_CUDA_TRY(cudaFreeAsync(arrived, stream));
    if (mind) FPH_CUDA_TRY(cudaFreeAsync(mind, stream));
    return FPH_OK;
}

}  // namespace fph
