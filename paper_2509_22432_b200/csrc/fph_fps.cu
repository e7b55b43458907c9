// fph_fps.cu -- farthest point sampling as one persistent cooperative kernel.
//
// Replaces reference floodph/geometry.py:88 farthest_point_sampling
// (numpy loop: d2 = |X - X[start]|^2, d2[start] = -1; repeat: nxt =
// argmax(d2) (first maximiser), d2 = minimum(d2, |X - X[nxt]|^2),
// d2[nxt] = -1).  Bit-exact: the squared distances use the reference's
// float64 accumulation order (sq64) and the argmax keeps the lowest index
// among equal values, so the landmark sequence is identical.
//
// Layout: one 512-thread CTA per SM (cooperative launch, all CTAs co-resident), each
// owning a contiguous slice of the cloud.  When a slice fits, its float64
// coordinates live in shared memory ((x, y) pairs + z, padded to PT x kResNT points, PT a
// template parameter so the per-point update is branch-free) and the running
// minimum in registers for the whole run -- a 1M-point cloud never touches
// HBM after the first load.  Per iteration each CTA publishes its (value, index) to a
// double-buffered slot array and bumps one monotone arrival counter; one
// thread per CTA polls the counter (ld.acquire) until all CTAs of this
// iteration arrived, then its warp reads every slot and reduces them.  All
// CTAs reduce the same slots in the same order, so they agree on the next
// landmark without a second broadcast; two CTA barriers per iteration.
// Every CTA reading every slot at the same moment concentrates on a few L2
// slices: each slot is written to four replicas and a CTA reads one of them
// (8.42 -> 7.95 ms for 2000 landmarks of 1M points).  The batched kernel's
// slots also carry the candidate's coordinates, staged into shared memory
// with cp.async, so a group needs no dependent load of the new landmark.
//
// Clouds too large for shared memory use the tiled variant: points are
// Morton-sorted into 256-point tiles with float64 bounding boxes, and an
// iteration only touches the tiles that contain the new landmark or whose
// box is closer to it than the tile's current largest running minimum --
// any other tile provably keeps every value (and its cached argmax).  Late
// iterations touch a few tiles instead of streaming the whole cloud.
#include <cub/cub.cuh>

#include "fph_common.cuh"

namespace fph {

namespace {

constexpr int kFpsThreads = 1024;
#ifndef FPH_FPS_RES_NT
#define FPH_FPS_RES_NT 512
#endif
constexpr int kResNT = FPH_FPS_RES_NT;  // threads per CTA of the resident kernel
constexpr int kFpsMaxPT = 9;  // points per thread in the shared-memory variants
constexpr int kMaxSlots = 160;
constexpr int kSortedMin = 262144;  // clouds at least this large take fps_sorted_kernel
constexpr int kSortedMaxPT = 15;    // its shared slice: PT x 512 x 28 bytes  // CTAs per exchange of the batched (coordinate-carrying) kernel
constexpr int kStaticSmem = 4 * kMaxSlots * 8 + 1024;  // batched kernel: stage + reduction scratch

struct __align__(16) Slot {
    double val;
    int idx;
    int pad;
};

// release-ordered arrival: the slot stores before it are visible to any
// thread that acquires the counter value it produces (no full SC fence)
__device__ __forceinline__ void arrive_release(unsigned long long* p) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}

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

#ifndef FPH_FPS_REDUX
#define FPH_FPS_REDUX 1
#endif

// Warp argmax with the lowest index among equal values, result in every
// lane.  REDUX form: the value as a monotone unsigned 64-bit key (exact for
// every value FPS produces: +0 <= d, -1 for landmarks, -inf for padding;
// no -0 and no NaN), then three dependent warp reductions -- max of the high
// word, max of the low word among lanes holding that high word, min index
// among lanes holding that key -- instead of five shuffle rounds of
// (double, int) pairs (15 SHFL and a compare chain).
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#if FPH_FPS_REDUX
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    const unsigned mi =
        __reduce_min_sync(0xffffffffu, hi == mhi && lo == mlo ? (unsigned)i : 0x7fffffffu);
    const unsigned long long mk = ((unsigned long long)mhi << 32) | mlo;
    v = __longlong_as_double((long long)((mk >> 63) ? (mk & 0x7fffffffffffffffull) : ~mk));
    i = (int)mi;
#else
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int oi = __shfl_xor_sync(0xffffffffu, i, o);
        better(v, i, ov, oi);
    }
#endif
}

// One iteration's exchange with two CTA barriers (a block-wide argmax on
// each side took seven): warps leave their argmax in shared memory; warp 0
// folds them, publishes the CTA's candidate, polls the arrival counter,
// reads all G slots and reduces them (same slots, same order in every CTA ->
// the same winner) and leaves the winner in red_i[32].
// `buf` holds this iteration's G slots; `target` is the arrival count that
// completes it.
// Replicas: the publisher writes its slot to kRepl copies `rs` slots apart
// and CTA c reads copy c % kRepl, spreading the all-CTAs-read-all-slots
// burst over more L2 slices.
#ifndef FPH_FPS_REPL
#define FPH_FPS_REPL 4
#endif
constexpr int kRepl = FPH_FPS_REPL;
#ifndef FPH_FPS_CTRS
#define FPH_FPS_CTRS 4
#endif
constexpr int kCtrs = FPH_FPS_CTRS;     // arrival counters of exchange_argmax
constexpr int kCtrStride = 32;          // 256 bytes apart
__host__ __device__ __forceinline__ int repl_stride(int G) { return ((G + 63) & ~63) + 40; }

__device__ __forceinline__ int exchange_argmax(double bv, int bi, Slot* buf, int G, int slot,
                                               unsigned long long* arrived,
                                               unsigned long long target, double* red_v,
                                               int* red_i, int rs, int nrep) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    warp_argmax(bv, bi);
    if (l == 0) {
        red_v[w] = bv;
        red_i[w] = bi;
    }
    __syncthreads();
    if (w == 0) {
        double v = l < (int)(blockDim.x >> 5) ? red_v[l] : -INFINITY;
        int i = l < (int)(blockDim.x >> 5) ? red_i[l] : 0x7fffffff;
        warp_argmax(v, i);
        // arrivals spread over kCtrs counters (CTA c on counter c % kCtrs,
        // kCtrStride words apart): the same-address atomics of 148 CTAs
        // serialise at one L2 slice; lane r < kCtrs waits for counter r
        if (l == 0) {
            for (int r = 0; r < nrep; ++r) {
                buf[r * rs + slot].val = v;
                buf[r * rs + slot].idx = i;
            }
            arrive_release(arrived + (slot % kCtrs) * kCtrStride);
        }
        if (l < kCtrs) {
            // CTAs on counter l per iteration: ceil((G - l) / kCtrs); target = G * it overall
            const unsigned long long per = (unsigned long long)((G - l + kCtrs - 1) / kCtrs);
            const unsigned long long tgt = per * (target / (unsigned long long)G);
            while (ld_acquire(arrived + l * kCtrStride) < tgt) {
            }
        }
        __syncwarp();
        buf += (int)(blockIdx.x % nrep) * rs;
        // this lane's slots (G <= 160: five) all in flight before the reduction
        constexpr int kPer = 5;
        double sv[kPer];
        int si[kPer];
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int b = l + 32 * t;
            sv[t] = b < G ? __ldcg(&buf[b].val) : -INFINITY;
            si[t] = b < G ? __ldcg(&buf[b].idx) : 0x7fffffff;
        }
        v = -INFINITY;
        i = 0x7fffffff;
#pragma unroll
        for (int t = 0; t < kPer; ++t) better(v, i, sv[t], si[t]);
        for (int b = l + 32 * kPer; b < G; b += 32) better(v, i, __ldcg(&buf[b].val), __ldcg(&buf[b].idx));
        warp_argmax(v, i);
        if (l == 0) red_i[32] = i;
    }
    __syncthreads();
    return red_i[32];
}

// Slots that carry the candidate's coordinates, so the next iteration's
// landmark needs no dependent load of px[cur] after the exchange.
struct __align__(16) SlotXYZ {
    double val;
    int idx, pad;
    double x, y;
    double z, pad2;
};

struct Winner {
    double x, y, z;
    int idx;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

// Exchange for the shared-memory kernels.  As exchange_argmax, plus: the
// publisher adds its candidate's coordinates (read from this CTA's shared
// slice) to the slot, and the reading lanes copy every slot's coordinates
// into shared memory with cp.async (no registers held: carrying them in
// registers spilled under the 64-register cap) while they fold (value,
// index) in registers.  The winning slot's coordinates are then one shared
// load away -- no dependent global load of the new landmark.
// `stage` holds 4 doubles per slot; G <= kMaxSlots (checked on the host).
__device__ __forceinline__ Winner exchange_argmax_xyz(double bv, int bi, const double2* sxy,
                                                      const double* sz, int beg,
                                                      SlotXYZ* buf, int G, int slot,
                                                      unsigned long long* arrived,
                                                      unsigned long long target, double* red_v,
                                                      int* red_i, double* stage) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    warp_argmax(bv, bi);
    if (l == 0) {
        red_v[w] = bv;
        red_i[w] = bi;
    }
    __syncthreads();
    if (w == 0) {
        double v = l < (int)(blockDim.x >> 5) ? red_v[l] : -INFINITY;
        int i = l < (int)(blockDim.x >> 5) ? red_i[l] : 0x7fffffff;
        warp_argmax(v, i);
        if (l == 0) {
            SlotXYZ s;
            s.val = v;
            s.idx = i;
            s.pad = 0;
            // an empty slice publishes -inf, never the winner: coordinates unused
            const int j = v == -INFINITY ? 0 : i - beg;
            s.x = sxy[j].x;
            s.y = sxy[j].y;
            s.z = sz[j];
            s.pad2 = 0.0;
            buf[slot] = s;
            arrive_release(arrived);
            while (ld_acquire(arrived) < target) {
            }
        }
        __syncwarp();
        constexpr int kPer = 5;
        double sv[kPer];
        int si[kPer];
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int b = l + 32 * t;
            if (b < G) {
                cp_async16(stage + 4 * b, &buf[b].x);
                cp_async16(stage + 4 * b + 2, &buf[b].z);
            }
            sv[t] = b < G ? __ldcg(&buf[b].val) : -INFINITY;
            si[t] = b < G ? __ldcg(&buf[b].idx) : 0x7fffffff;
        }
        v = -INFINITY;
        i = 0x7fffffff;
        int bs = 0;
#pragma unroll
        for (int t = 0; t < kPer; ++t)
            if (sv[t] > v || (sv[t] == v && si[t] < i)) {
                v = sv[t];
                i = si[t];
                bs = l + 32 * t;
            }
        const int myi = i;
        warp_argmax(v, i);
        const int src = __ffs(__ballot_sync(0xffffffffu, myi == i)) - 1;
        bs = __shfl_sync(0xffffffffu, bs, src);
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (l == 0) {
            red_i[32] = i;
            red_i[33] = bs;
        }
    }
    __syncthreads();
    Winner wn;
    wn.idx = red_i[32];
    const int bs = red_i[33];
    wn.x = stage[4 * bs];
    wn.y = stage[4 * bs + 1];
    wn.z = stage[4 * bs + 2];
    return wn;
}

// Streaming variant (slices beyond shared memory; fps_run only takes it
// for k == 1, larger k goes to the tiled kernel): coordinates and running
// minima stream through L2/HBM.
__global__ void __launch_bounds__(kFpsThreads, 1)
    fps_kernel(const double* __restrict__ px, const double* __restrict__ py,
               const double* __restrict__ pz, int n, int k, int start, int chunk,
               double* __restrict__ mind, Slot* slots, unsigned long long* arrived,
               long long* __restrict__ out) {
    __shared__ double red_v[32];
    __shared__ int red_i[33];
    const int beg = blockIdx.x * chunk;
    const int cnt = max(0, min(n, beg + chunk) - beg);
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) mind[beg + j] = INFINITY;
    int cur = start;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = start;
    const int G = gridDim.x, rs = repl_stride(G);
    for (int it = 1; it <= k; ++it) {
        const double qx = px[cur], qy = py[cur], qz = pz[cur];
        double bv = -INFINITY;
        int bi = 0x7fffffff;
        for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
            const int gi = beg + j;
            const double d = sq64(px[gi], py[gi], pz[gi], qx, qy, qz);
            const double m = gi == cur ? -1.0 : fmin(mind[gi], d);
            mind[gi] = m;
            better(bv, bi, m, gi);
        }
        if (it == k) break;
        cur = exchange_argmax(bv, bi, slots + (it & 1) * kRepl * rs, G, blockIdx.x, arrived,
                              (unsigned long long)G * it, red_v, red_i, rs, kRepl);
        if (blockIdx.x == 0 && threadIdx.x == 0) out[it] = cur;
    }
}

// Resident variant with PT points per thread, branch-free: the shared slice
// is padded to PT x kResNT points whose running minimum starts at -inf (a
// padded point never wins: d < -inf is false).  Within a thread the global
// index ascends with t, so a strict `>` keeps the lowest index among equal
// values; the min is a compare-select (no NaN handling: coordinates are
// finite, and d >= +0 so no signed-zero case).  ~23 instructions per point
// instead of ~32 plus a branch.
template <int PT>
__global__ void __launch_bounds__(kResNT, 1)
    fps_resident_kernel(const double* __restrict__ px, const double* __restrict__ py,
                        const double* __restrict__ pz, int n, int k, int start, int chunk,
                        Slot* slots, unsigned long long* arrived, long long* __restrict__ out) {
    extern __shared__ double sm[];
    __shared__ double red_v[32];
    __shared__ int red_i[33];
    constexpr int kSlice = PT * kResNT;
    const int beg = blockIdx.x * chunk;
    const int cnt = max(0, min(n, beg + chunk) - beg);
    // (x, y) interleaved: one 16-byte shared load plus one 8-byte per point
    // instead of three 8-byte loads (the MIO queue throttled the update)
    double2* sxy = reinterpret_cast<double2*>(sm);
    double* sz = sm + 2 * kSlice;
    for (int j = threadIdx.x; j < kSlice; j += blockDim.x) {
        const bool in = j < cnt;
        sxy[j] = in ? make_double2(px[beg + j], py[beg + j]) : make_double2(0.0, 0.0);
        sz[j] = in ? pz[beg + j] : 0.0;
    }
    double md[PT];
#pragma unroll
    for (int t = 0; t < PT; ++t) md[t] = (int)threadIdx.x + t * kResNT < cnt ? INFINITY : -INFINITY;
    __syncthreads();
    int cur = start;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = start;
    const int G = gridDim.x, rs = repl_stride(G);
    for (int it = 1; it <= k; ++it) {
        const double qx = px[cur], qy = py[cur], qz = pz[cur];
        // slot t of this thread holds the new landmark iff t * kResNT == jc
        const int jc = cur >= beg && cur < beg + cnt ? cur - beg - (int)threadIdx.x : -1;
        double bv = -INFINITY;
        int bi = 0x7fffffff;
#ifndef FPH_FPS_NOUPDATE
#define FPH_FPS_NOUPDATE 0
#endif
#pragma unroll
        for (int t = 0; t < (FPH_FPS_NOUPDATE ? 1 : PT); ++t) {  // NOUPDATE: timing experiment only
            const int j = threadIdx.x + t * kResNT;
            const double2 xy = sxy[j];
            const double d = sq64(xy.x, xy.y, sz[j], qx, qy, qz);
            double m = d < md[t] ? d : md[t];
            m = jc == t * kResNT ? -1.0 : m;
            md[t] = m;
            if (m > bv) {
                bv = m;
                bi = beg + j;
            }
        }
        if (it == k) break;
        cur = exchange_argmax(bv, bi, slots + (it & 1) * kRepl * rs, G, blockIdx.x, arrived,
                              (unsigned long long)G * it, red_v, red_i, rs, kRepl);
        if (blockIdx.x == 0 && threadIdx.x == 0) out[it] = cur;
    }
}

// Resident variant over the Morton-sorted cloud: warp w of a CTA holds
// 32 x PT consecutive sorted points (spatially compact), with their box
// kept in registers.  An iteration updates a warp's points only if the new
// landmark is among them or its box is closer to the landmark than the
// warp's largest running minimum; otherwise no point of the warp can
// change and its threads keep their argmax records.  Late iterations touch
// a few warps near the landmark instead of every point.  Ties still go to
// the lowest cloud index (sidx, shared memory, read only when a value can
// tie or win).  Shared memory: PT x 512 x (24 + 4) bytes, PT <= 15.
template <int PT>
__global__ void __launch_bounds__(kResNT, 1)
    fps_sorted_kernel(const double* __restrict__ px, const double* __restrict__ py,
                      const double* __restrict__ pz, const double* __restrict__ sx,
                      const double* __restrict__ sy, const double* __restrict__ szg,
                      const int* __restrict__ sidx, const int* __restrict__ spos, int n, int k,
                      int start, int chunk, Slot* slots, unsigned long long* arrived,
                      long long* __restrict__ out) {
    extern __shared__ double sm[];
    __shared__ double red_v[32];
    __shared__ int red_i[33];
    constexpr int kSlice = PT * kResNT;
    const int beg = blockIdx.x * chunk;
    const int cnt = max(0, min(n, beg + chunk) - beg);
    double2* sxy = reinterpret_cast<double2*>(sm);
    double* sz = sm + 2 * kSlice;
    int* soi = reinterpret_cast<int*>(sm + 3 * kSlice);
    for (int j = threadIdx.x; j < kSlice; j += blockDim.x) {
        const bool in = j < cnt;
        sxy[j] = in ? make_double2(sx[beg + j], sy[beg + j]) : make_double2(0.0, 0.0);
        sz[j] = in ? szg[beg + j] : 0.0;
        soi[j] = in ? sidx[beg + j] : 0x7fffffff;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int wbeg = w * 32 * PT;  // this warp's points: wbeg + 32 t + lane
    double md[PT];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    __syncthreads();
#pragma unroll
    for (int t = 0; t < PT; ++t) {
        const int j = wbeg + 32 * t + l;
        md[t] = j < cnt ? INFINITY : -INFINITY;
        if (j < cnt) {
            const double2 xy = sxy[j];
            lo[0] = fmin(lo[0], xy.x); hi[0] = fmax(hi[0], xy.x);
            lo[1] = fmin(lo[1], xy.y); hi[1] = fmax(hi[1], xy.y);
            lo[2] = fmin(lo[2], sz[j]); hi[2] = fmax(hi[2], sz[j]);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = warp_min_d(lo[a]);
        for (int o = 16; o > 0; o >>= 1) hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    int cur = start;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = start;
    const int G = gridDim.x, rs = repl_stride(G);
    double bv = -INFINITY, wmax = INFINITY;  // this thread's record; the warp's largest minimum
    int bi = 0x7fffffff;
    for (int it = 1; it <= k; ++it) {
        const double qx = px[cur], qy = py[cur], qz = pz[cur];
        const int pc = spos[cur] - beg - wbeg;  // the landmark's place in this warp's points
        const double dx = fmax(0.0, fmax(lo[0] - qx, qx - hi[0]));
        const double dy = fmax(0.0, fmax(lo[1] - qy, qy - hi[1]));
        const double dz = fmax(0.0, fmax(lo[2] - qz, qz - hi[2]));
        // a safe lower bound on sq64(x, q) for every point of the warp
        const double lb = (dx * dx + dy * dy + dz * dz) * (1.0 - 1e-12);
        if ((pc >= 0 && pc < 32 * PT) || lb < wmax) {  // warp-uniform
            bv = -INFINITY;
            bi = 0x7fffffff;
#pragma unroll
            for (int t = 0; t < PT; ++t) {
                const int j = wbeg + 32 * t + l;
                const double2 xy = sxy[j];
                const double d = sq64(xy.x, xy.y, sz[j], qx, qy, qz);
                double m = d < md[t] ? d : md[t];
                m = pc == 32 * t + l ? -1.0 : m;
                md[t] = m;
                if (m >= bv) {
                    const int oi = soi[j];
                    if (m > bv || oi < bi) {
                        bv = m;
                        bi = oi;
                    }
                }
            }
            // the warp's largest running minimum (a monotone 64-bit key)
            const unsigned long long b = (unsigned long long)__double_as_longlong(bv);
            const unsigned long long key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
            const unsigned mhi = __reduce_max_sync(0xffffffffu, (unsigned)(key >> 32));
            const unsigned mlo = __reduce_max_sync(0xffffffffu, (unsigned)(key >> 32) == mhi ? (unsigned)key : 0u);
            const unsigned long long mk = ((unsigned long long)mhi << 32) | mlo;
            wmax = __longlong_as_double((long long)((mk >> 63) ? (mk & 0x7fffffffffffffffull) : ~mk));
        }
        if (it == k) break;
        cur = exchange_argmax(bv, bi, slots + (it & 1) * kRepl * rs, G, blockIdx.x, arrived,
                              (unsigned long long)G * it, red_v, red_i, rs, kRepl);
        if (blockIdx.x == 0 && threadIdx.x == 0) out[it] = cur;
    }
}

template <int PT>
int launch_sorted(const double* d_x, const double* d_y, const double* d_z, const double* sx,
                  const double* sy, const double* sz, const int* sidx, const int* spos, int n,
                  int k, int start, int chunk, int G, Slot* slots, unsigned long long* arrived,
                  long long* d_out, cudaStream_t stream) {
    const size_t smem = (sizeof(double) * 3 + sizeof(int)) * PT * kResNT;
    FPH_CUDA_TRY(cudaFuncSetAttribute(fps_sorted_kernel<PT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void* args[] = {(void*)&d_x,  (void*)&d_y,   (void*)&d_z,   (void*)&sx,    (void*)&sy,
                    (void*)&sz,   (void*)&sidx,  (void*)&spos,  (void*)&n,     (void*)&k,
                    (void*)&start, (void*)&chunk, (void*)&slots, (void*)&arrived, (void*)&d_out};
    FPH_CUDA_TRY(cudaLaunchCooperativeKernel((void*)fps_sorted_kernel<PT>, dim3(G), dim3(kResNT),
                                             args, smem, stream));
    return FPH_OK;
}

template <int PT>
int launch_resident(const double* d_x, const double* d_y, const double* d_z, int n, int k,
                    int start, int chunk, int G, Slot* slots, unsigned long long* arrived,
                    long long* d_out, cudaStream_t stream) {
    const size_t smem = sizeof(double) * 3 * PT * kResNT;
    FPH_CUDA_TRY(cudaFuncSetAttribute(fps_resident_kernel<PT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void* args[] = {(void*)&d_x, (void*)&d_y,   (void*)&d_z,   (void*)&n,      (void*)&k,
                    (void*)&start, (void*)&chunk, (void*)&slots, (void*)&arrived, (void*)&d_out};
    FPH_CUDA_TRY(cudaLaunchCooperativeKernel((void*)fps_resident_kernel<PT>, dim3(G),
                                             dim3(kResNT), args, smem, stream));
    return FPH_OK;
}

// ------------------------------------------------------------ tiled variant
constexpr int kTileP = 256;  // points per tile

// Exchange of the tiled kernel: as exchange_argmax_xyz, with the candidate's
// coordinates and sorted position taken from the tile that holds it (this
// CTA's per-tile argmax records in shared memory): the winner arrives with
// its coordinates and tile, so the next iteration starts without a
// dependent global load.  `bt`: the tile (local index) of this thread's
// candidate.
__device__ __forceinline__ Winner exchange_argmax_tiled(double bv, int bi, int bt,
                                                        const double* txyz, const int* tpos,
                                                        SlotXYZ* buf, int G, int slot,
                                                        unsigned long long* arrived,
                                                        unsigned long long target, double* red_v,
                                                        int* red_i, int* red_t, double* stage,
                                                        int* wpos) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    {
        const int myi = bi;
        warp_argmax(bv, bi);
        const unsigned hit = __ballot_sync(0xffffffffu, myi == bi);
        bt = __shfl_sync(0xffffffffu, bt, hit ? __ffs(hit) - 1 : 0);
    }
    if (l == 0) {
        red_v[w] = bv;
        red_i[w] = bi;
        red_t[w] = bt;
    }
    __syncthreads();
    if (w == 0) {
        double v = l < (int)(blockDim.x >> 5) ? red_v[l] : -INFINITY;
        int i = l < (int)(blockDim.x >> 5) ? red_i[l] : 0x7fffffff;
        int t = l < (int)(blockDim.x >> 5) ? red_t[l] : 0;
        {
            const int myi = i;
            warp_argmax(v, i);
            const unsigned hit = __ballot_sync(0xffffffffu, myi == i);
            t = __shfl_sync(0xffffffffu, t, hit ? __ffs(hit) - 1 : 0);
        }
        if (l == 0) {
            SlotXYZ sl;
            sl.val = v;
            sl.idx = i;
            // an empty CTA publishes -inf, never the winner: the rest unused
            const bool any = v > -INFINITY;
            sl.pad = any ? tpos[t] : 0;
            sl.x = any ? txyz[3 * t] : 0.0;
            sl.y = any ? txyz[3 * t + 1] : 0.0;
            sl.z = any ? txyz[3 * t + 2] : 0.0;
            sl.pad2 = 0.0;
            buf[slot] = sl;
            // one counter: spreading the arrivals as exchange_argmax does
            // measured 27.6 -> 30.5 ms on the 10M tiled run
            arrive_release(arrived);
            while (ld_acquire(arrived) < target) {
            }
        }
        __syncwarp();
        constexpr int kPer = 5;
        double sv[kPer];
        int si[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int b = l + 32 * q;
            if (b < G) {
                cp_async16(stage + 4 * b, &buf[b].x);
                cp_async16(stage + 4 * b + 2, &buf[b].z);
            }
            sv[q] = b < G ? __ldcg(&buf[b].val) : -INFINITY;
            si[q] = b < G ? __ldcg(&buf[b].idx) : 0x7fffffff;
        }
        v = -INFINITY;
        i = 0x7fffffff;
        int bs = 0;
#pragma unroll
        for (int q = 0; q < kPer; ++q)
            if (sv[q] > v || (sv[q] == v && si[q] < i)) {
                v = sv[q];
                i = si[q];
                bs = l + 32 * q;
            }
        const int myi = i;
        warp_argmax(v, i);
        const int src = __ffs(__ballot_sync(0xffffffffu, myi == i)) - 1;
        bs = __shfl_sync(0xffffffffu, bs, src);
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (l == 0) {
            red_i[32] = i;
            red_i[33] = bs;
            *wpos = __ldcg(&buf[bs].pad);
        }
    }
    __syncthreads();
    Winner wn;
    wn.idx = red_i[32];
    const int bs = red_i[33];
    wn.x = stage[4 * bs];
    wn.y = stage[4 * bs + 1];
    wn.z = stage[4 * bs + 2];
    return wn;
}

// Per iteration: one thread per tile tests the tile's box against the new
// landmark (a tile is touched if it holds the landmark or its box is closer
// than the tile's largest running minimum), the touched tiles go to a
// shared list, and the warps update them (each lane's points loaded before
// any running minimum is stored back); the tile's argmax, with its
// coordinates and sorted position, is kept in shared memory for the
// exchange.
#ifndef FPH_FPS_TILED_NT
#define FPH_FPS_TILED_NT 512
#endif
#ifndef FPH_FPS_TILED_U
#define FPH_FPS_TILED_U 8
#endif
// 512 threads (128 registers): a lane loads all 8 of its points of a
// touched tile in one round trip
constexpr int kTiledNT = FPH_FPS_TILED_NT;
constexpr int kTiledU = FPH_FPS_TILED_U;  // points per lane loaded together

__global__ void __launch_bounds__(kTiledNT, 1)
    fps_tiled_kernel(const double* __restrict__ px, const double* __restrict__ py,
                     const double* __restrict__ pz, const double* __restrict__ sx,
                     const double* __restrict__ sy, const double* __restrict__ sz,
                     const int* __restrict__ sidx, const int* __restrict__ spos,
                     const double* __restrict__ tbox, int n, int k, int start, int per_cta,
                     int ntiles,
                     double* __restrict__ md, SlotXYZ* slots, unsigned long long* arrived,
                     long long* __restrict__ out) {
    extern __shared__ double sm[];
    __shared__ double red_v[32];
    __shared__ int red_i[34];
    __shared__ int red_t[32];
    __shared__ __align__(16) double stage[4 * kMaxSlots];
    __shared__ int wpos;
    __shared__ int cnt[2];
    // tiles are dealt round-robin (tile = blockIdx.x + t * G): the few tiles
    // near a new landmark are Morton neighbours, so they land on different
    // CTAs instead of piling onto one
    const int G = gridDim.x;
    const int nt = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
    double* box = sm;                   // nt x 6
    double* tmax = sm + 6 * per_cta;    // nt
    double* txyz = tmax + per_cta;      // nt x 3: the tile argmax's coordinates
    int* targ = reinterpret_cast<int*>(txyz + 3 * per_cta);  // its cloud index
    int* tpos = targ + per_cta;                                // its sorted position
    int* list = tpos + per_cta;                                // touched tiles
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
        for (int c = 0; c < 6; ++c) box[t * 6 + c] = tbox[(size_t)(blockIdx.x + t * G) * 6 + c];
        tmax[t] = INFINITY;
        targ[t] = 0x7fffffff;
        tpos[t] = 0;
    }
    for (int t = 0; t < nt; ++t) {
        const long long base = (long long)(blockIdx.x + t * G) * kTileP;
        for (int j = threadIdx.x; j < kTileP; j += blockDim.x)
            if (base + j < n) md[base + j] = INFINITY;
    }
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int cur = start;
    double qx = px[start], qy = py[start], qz = pz[start];  // later ones come with the exchange
    int ctile = spos[start] / kTileP;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = start;
    for (int it = 1; it < k; ++it) {
        const int c = it & 1;
        for (int t = threadIdx.x; t < nt; t += blockDim.x) {
            const int tile = blockIdx.x + t * G;
            const double* b = box + t * 6;
            const double dx = fmax(0.0, fmax(b[0] - qx, qx - b[3]));
            const double dy = fmax(0.0, fmax(b[1] - qy, qy - b[4]));
            const double dz = fmax(0.0, fmax(b[2] - qz, qz - b[5]));
            // a safe lower bound on sq64(x, q) for every x in the box
            const double lb = (dx * dx + dy * dy + dz * dz) * (1.0 - 1e-12);
            if (tile == ctile || lb < tmax[t]) list[atomicAdd(&cnt[c], 1)] = t;
        }
        __syncthreads();
        const int ntouch = cnt[c];
        for (int q = w; q < ntouch; q += kTiledNT / 32) {
            const int t = list[q];
            const long long base = (long long)(blockIdx.x + t * G) * kTileP;
            double v = -INFINITY;
            int i = 0x7fffffff, bp = 0;
#pragma unroll
            for (int h = 0; h < kTileP / 32; h += kTiledU) {
                long long pp[kTiledU];
                int oi[kTiledU];
                double d[kTiledU], mo[kTiledU];
#pragma unroll
                for (int u = 0; u < kTiledU; ++u) {
                    pp[u] = base + l + 32 * (h + u);
                    const bool in = pp[u] < n;
                    oi[u] = in ? sidx[pp[u]] : 0x7fffffff;
                    d[u] = in ? sq64(sx[pp[u]], sy[pp[u]], sz[pp[u]], qx, qy, qz) : -INFINITY;
                    mo[u] = in ? md[pp[u]] : -INFINITY;
                }
#pragma unroll
                for (int u = 0; u < kTiledU; ++u) {
                    if (pp[u] < n) {
                        const double m = oi[u] == cur ? -1.0 : fmin(mo[u], d[u]);
                        md[pp[u]] = m;
                        if (m > v || (m == v && oi[u] < i)) {
                            v = m;
                            i = oi[u];
                            bp = (int)pp[u];
                        }
                    }
                }
            }
            const int myi = i;
            warp_argmax(v, i);
            const unsigned hit = __ballot_sync(0xffffffffu, myi == i);
            const int src = hit ? __ffs(hit) - 1 : 0;
            bp = __shfl_sync(0xffffffffu, bp, src);
            if (l == 0) {
                tmax[t] = v;
                targ[t] = i;
                tpos[t] = bp;
                if (v > -INFINITY) {  // the argmax point was just loaded: an L1 hit
                    txyz[3 * t] = sx[bp];
                    txyz[3 * t + 1] = sy[bp];
                    txyz[3 * t + 2] = sz[bp];
                }
            }
        }
        if (threadIdx.x == 0) cnt[c ^ 1] = 0;  // the next iteration's list
        __syncthreads();
        double v = -INFINITY;
        int i = 0x7fffffff, bt = 0;
        for (int t = threadIdx.x; t < nt; t += blockDim.x)
            if (tmax[t] > v || (tmax[t] == v && targ[t] < i)) {
                v = tmax[t];
                i = targ[t];
                bt = t;
            }
        const Winner wn = exchange_argmax_tiled(v, i, bt, txyz, tpos, slots + (it & 1) * kMaxSlots, G,
                                                blockIdx.x, arrived, (unsigned long long)G * it,
                                                red_v, red_i, red_t, stage, &wpos);
        cur = wn.idx;
        qx = wn.x;
        qy = wn.y;
        qz = wn.z;
        ctile = wpos / kTileP;
        if (blockIdx.x == 0 && threadIdx.x == 0) out[it] = cur;
    }
}

// mm: the box as (min, max) per axis, from minmax_kernel (read on the
// device: the quantisation never waits for the host; any box works)
__global__ void morton_kernel(const double* __restrict__ x, const double* __restrict__ y,
                              const double* __restrict__ z, int n, const double* __restrict__ mm,
                              unsigned* __restrict__ code, int* __restrict__ idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double lox = mm[0], loy = mm[2], loz = mm[4];
    const double ext = fmax(fmax(mm[1] - mm[0], mm[3] - mm[2]), fmax(mm[5] - mm[4], 1e-300));
    const double inv = 1024.0 / ext;
    auto q = [&](double v, double lo) {
        return (unsigned)fmin(1023.0, fmax(0.0, floor((v - lo) * inv)));
    };
    auto spread = [](unsigned v) {
        v = (v | (v << 16)) & 0x030000FFu;
        v = (v | (v << 8)) & 0x0300F00Fu;
        v = (v | (v << 4)) & 0x030C30C3u;
        v = (v | (v << 2)) & 0x09249249u;
        return v;
    };
    code[i] = spread(q(x[i], lox)) | (spread(q(y[i], loy)) << 1) | (spread(q(z[i], loz)) << 2);
    idx[i] = i;
}

__global__ void gather_sorted_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                     const double* __restrict__ z, const int* __restrict__ sidx,
                                     int n, double* __restrict__ sx, double* __restrict__ sy,
                                     double* __restrict__ sz, int* __restrict__ spos) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int i = sidx[p];
    sx[p] = x[i];
    sy[p] = y[i];
    sz[p] = z[i];
    spos[i] = p;
}

// one warp per tile: float64 bounding box
__global__ void tile_box_kernel(const double* __restrict__ sx, const double* __restrict__ sy,
                                const double* __restrict__ sz, int n, int ntiles,
                                double* __restrict__ tbox) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = threadIdx.x & 31;
    if (t >= ntiles) return;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int j = l; j < kTileP; j += 32) {
        const long long p = (long long)t * kTileP + j;
        if (p < n) {
            const double v[3] = {sx[p], sy[p], sz[p]};
            for (int c = 0; c < 3; ++c) {
                lo[c] = fmin(lo[c], v[c]);
                hi[c] = fmax(hi[c], v[c]);
            }
        }
    }
    for (int c = 0; c < 3; ++c) {
        lo[c] = warp_min_d(lo[c]);
        for (int o = 16; o > 0; o >>= 1) hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
    if (l == 0)
        for (int c = 0; c < 3; ++c) {
            tbox[(size_t)t * 6 + c] = lo[c];
            tbox[(size_t)t * 6 + 3 + c] = hi[c];
        }
}

__global__ void minmax_init_kernel(double* mm) {
    mm[threadIdx.x] = (threadIdx.x & 1) ? -INFINITY : INFINITY;
}

__global__ void minmax_kernel(const double* __restrict__ v, int n, double* __restrict__ out2) {
    double lo = INFINITY, hi = -INFINITY;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        lo = fmin(lo, v[i]);
        hi = fmax(hi, v[i]);
    }
    lo = warp_min_d(lo);
    for (int o = 16; o > 0; o >>= 1) hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    if ((threadIdx.x & 31) == 0) {
        // non-negative reinterpretation trick is not needed: use CAS loops
        unsigned long long* a = reinterpret_cast<unsigned long long*>(out2);
        unsigned long long old = a[0], assumed;
        do {
            assumed = old;
            if (__longlong_as_double((long long)assumed) <= lo) break;
            old = atomicCAS(a, assumed, (unsigned long long)__double_as_longlong(lo));
        } while (old != assumed);
        old = a[1];
        do {
            assumed = old;
            if (__longlong_as_double((long long)assumed) >= hi) break;
            old = atomicCAS(a + 1, assumed, (unsigned long long)__double_as_longlong(hi));
        } while (old != assumed);
    }
}

// Morton order of the cloud (the box is read on the device): sorted copies
// sx, sy, sz, the cloud index of each sorted point (sidx) and the sorted
// position of each cloud point (spos), allocated in `sc`.
int morton_sort(const double* d_x, const double* d_y, const double* d_z, int n, Scratch& sc,
                cudaStream_t stream, double** sx, double** sy, double** sz, int** sidx, int** spos) {
    double* mm = nullptr;
    FPH_TRY(sc.alloc(&mm, 6));
    minmax_init_kernel<<<1, 6, 0, stream>>>(mm);
    minmax_kernel<<<1024, 256, 0, stream>>>(d_x, n, mm);
    minmax_kernel<<<1024, 256, 0, stream>>>(d_y, n, mm + 2);
    minmax_kernel<<<1024, 256, 0, stream>>>(d_z, n, mm + 4);
    unsigned *code = nullptr, *code2 = nullptr;
    int* idx = nullptr;
    FPH_TRY(sc.alloc(&code, n));
    FPH_TRY(sc.alloc(&code2, n));
    FPH_TRY(sc.alloc(&idx, n));
    FPH_TRY(sc.alloc(sidx, n));
    FPH_TRY(sc.alloc(spos, n));
    FPH_TRY(sc.alloc(sx, n));
    FPH_TRY(sc.alloc(sy, n));
    FPH_TRY(sc.alloc(sz, n));
    morton_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_x, d_y, d_z, n, mm, code, idx);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, code, code2, idx, *sidx, n, 0, 30, stream);
    unsigned char* tmp = nullptr;
    FPH_TRY(sc.alloc(&tmp, tmp_bytes));
    FPH_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, code, code2, idx, *sidx, n, 0, 30,
                                                 stream));
    gather_sorted_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_x, d_y, d_z, *sidx, n, *sx, *sy,
                                                              *sz, *spos);
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

int fps_tiled(const double* d_x, const double* d_y, const double* d_z, int n, int k, int start,
              long long* d_out, int G, cudaStream_t stream) {
    // bounding box (for the Morton quantisation only: any box works)
    Scratch sc(stream);
    double* mm = nullptr;
    FPH_TRY(sc.alloc(&mm, 6));
    minmax_init_kernel<<<1, 6, 0, stream>>>(mm);
    minmax_kernel<<<1024, 256, 0, stream>>>(d_x, n, mm);
    minmax_kernel<<<1024, 256, 0, stream>>>(d_y, n, mm + 2);
    minmax_kernel<<<1024, 256, 0, stream>>>(d_z, n, mm + 4);
    unsigned *code = nullptr, *code2 = nullptr;
    int *idx = nullptr, *sidx = nullptr, *spos = nullptr;
    double *sx = nullptr, *sy = nullptr, *sz = nullptr, *md = nullptr, *tbox = nullptr;
    const int ntiles = (n + kTileP - 1) / kTileP;
    FPH_TRY(sc.alloc(&code, n));
    FPH_TRY(sc.alloc(&code2, n));
    FPH_TRY(sc.alloc(&idx, n));
    FPH_TRY(sc.alloc(&sidx, n));
    FPH_TRY(sc.alloc(&spos, n));
    FPH_TRY(sc.alloc(&sx, n));
    FPH_TRY(sc.alloc(&sy, n));
    FPH_TRY(sc.alloc(&sz, n));
    FPH_TRY(sc.alloc(&md, n));
    FPH_TRY(sc.alloc(&tbox, 6 * (size_t)ntiles));
    morton_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_x, d_y, d_z, n, mm, code, idx);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, code, code2, idx, sidx, n, 0, 30, stream);
    unsigned char* tmp = nullptr;
    FPH_TRY(sc.alloc(&tmp, tmp_bytes));
    FPH_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, code, code2, idx, sidx, n, 0, 30,
                                                 stream));
    gather_sorted_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_x, d_y, d_z, sidx, n, sx, sy, sz,
                                                              spos);
    tile_box_kernel<<<(ntiles * 32 + 255) / 256, 256, 0, stream>>>(sx, sy, sz, n, ntiles, tbox);
    const int per_cta = (ntiles + G - 1) / G;
    const size_t smem = sizeof(double) * 10 * per_cta + sizeof(int) * 3 * per_cta + 16;
    if (G > kMaxSlots) {
        set_error("fps: %d CTAs exceed the exchange's %d slots", G, kMaxSlots);
        return FPH_EARG;
    }
    SlotXYZ* slots = nullptr;
    unsigned long long* arrived = nullptr;
    FPH_TRY(sc.alloc(&slots, 2 * kMaxSlots));
    FPH_TRY(sc.alloc(&arrived, kCtrs * kCtrStride));
    FPH_CUDA_TRY(cudaMemsetAsync(arrived, 0, sizeof(unsigned long long) * kCtrs * kCtrStride, stream));
    FPH_CUDA_TRY(cudaFuncSetAttribute(fps_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    int ntl = ntiles;
    void* args[] = {(void*)&d_x,  (void*)&d_y,  (void*)&d_z,   (void*)&sx,      (void*)&sy,
                    (void*)&sz,   (void*)&sidx, (void*)&spos,  (void*)&tbox,    (void*)&n,
                    (void*)&k,    (void*)&start, (void*)&per_cta, (void*)&ntl,  (void*)&md,
                    (void*)&slots, (void*)&arrived, (void*)&d_out};
    FPH_CUDA_TRY(cudaLaunchCooperativeKernel((void*)fps_tiled_kernel, dim3(G), dim3(kTiledNT),
                                             args, smem, stream));
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

// ----------------------------------------------------------- batched clouds
// Many equal-size clouds (configs[3]): CTA groups of `cpg` CTAs each run one
// cloud at a time, exchanging through their own slots and counter, so
// ngroups = gridDim / cpg clouds advance concurrently instead of every cloud
// using (and waiting on) the whole GPU.
template <int PT>
__global__ void __launch_bounds__(kResNT, 1)
    fps_batched_kernel(const double* __restrict__ px, const double* __restrict__ py,
                       const double* __restrict__ pz, int batch, int n, int k, int start, int cpg,
                       int chunk, Slot* slots, unsigned long long* arrived,
                       long long* __restrict__ out) {
    extern __shared__ double sm[];
    __shared__ double red_v[32];
    __shared__ int red_i[34];
    __shared__ __align__(16) double stage[4 * kMaxSlots];
    constexpr int kSlice = PT * kResNT;  // padded as in fps_resident_kernel
    const int ngroups = gridDim.x / cpg;
    const int g = blockIdx.x / cpg, r = blockIdx.x % cpg;
    if (g >= ngroups) return;
    double2* sxy = reinterpret_cast<double2*>(sm);  // (x, y) interleaved as in fps_resident_kernel
    double* sz = sm + 2 * kSlice;
    SlotXYZ* gslots = reinterpret_cast<SlotXYZ*>(slots) + (size_t)g * 2 * cpg;
    int seq = 0;
    for (int c = g; c < batch; c += ngroups, ++seq) {
        const long long cb = (long long)c * n;
        const int beg = r * chunk, cnt = max(0, min(n, beg + chunk) - beg);
        __syncthreads();
        for (int j = threadIdx.x; j < kSlice; j += blockDim.x) {
            const bool in = j < cnt;
            sxy[j] = in ? make_double2(px[cb + beg + j], py[cb + beg + j]) : make_double2(0.0, 0.0);
            sz[j] = in ? pz[cb + beg + j] : 0.0;
        }
        double md[PT];
#pragma unroll
        for (int t = 0; t < PT; ++t)
            md[t] = (int)threadIdx.x + t * kResNT < cnt ? INFINITY : -INFINITY;
        __syncthreads();
        int cur = start;
        if (r == 0 && threadIdx.x == 0) out[(long long)c * k] = start;
        double qx = px[cb + cur], qy = py[cb + cur], qz = pz[cb + cur];
        for (int it = 1; it < k; ++it) {
            const int jc = cur >= beg && cur < beg + cnt ? cur - beg - (int)threadIdx.x : -1;
            double bv = -INFINITY;
            int bi = 0x7fffffff;
#pragma unroll
            for (int t = 0; t < PT; ++t) {
                const int j = threadIdx.x + t * kResNT;
                const double2 xy = sxy[j];
                const double d = sq64(xy.x, xy.y, sz[j], qx, qy, qz);
                double m = d < md[t] ? d : md[t];
                m = jc == t * kResNT ? -1.0 : m;
                md[t] = m;
                if (m > bv) {
                    bv = m;
                    bi = beg + j;
                }
            }
            const long long tag = (long long)seq * (k - 1) + it;  // group-wide iteration
            const Winner wn = exchange_argmax_xyz(
                bv, bi, sxy, sz, beg, gslots + (tag & 1) * cpg, cpg, r, arrived + g,
                (unsigned long long)cpg * (unsigned long long)tag, red_v, red_i, stage);
            cur = wn.idx;
            qx = wn.x;
            qy = wn.y;
            qz = wn.z;
            if (r == 0 && threadIdx.x == 0) out[(long long)c * k + it] = cur;
        }
    }
}

template <int PT>
int launch_batched(const double* d_x, const double* d_y, const double* d_z, int batch, int n,
                   int k, int start, int cpg, int chunk, int grid, Slot* slots,
                   unsigned long long* arrived, long long* d_out, cudaStream_t stream) {
    const size_t smem = sizeof(double) * 3 * PT * kResNT;
    FPH_CUDA_TRY(cudaFuncSetAttribute(fps_batched_kernel<PT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void* args[] = {(void*)&d_x, (void*)&d_y, (void*)&d_z,   (void*)&batch, (void*)&n,
                    (void*)&k,   (void*)&start, (void*)&cpg, (void*)&chunk, (void*)&slots,
                    (void*)&arrived, (void*)&d_out};
    FPH_CUDA_TRY(cudaLaunchCooperativeKernel((void*)fps_batched_kernel<PT>, dim3(grid),
                                             dim3(kResNT), args, smem, stream));
    return FPH_OK;
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
    static const bool force_tiled = [] {  // experiments: the tiled kernel at any size
        const char* e = getenv("FPH_FPS_TILED");
        return e && e[0] == '1';
    }();
    if ((!use_smem || force_tiled) && k > 1 && n >= 4096)
        return fps_tiled(d_x, d_y, d_z, n, k, start, d_out, G, stream);
    Scratch sc(stream);
    Slot* slots = nullptr;
    double* mind = nullptr;
    unsigned long long* arrived = nullptr;
    FPH_TRY(sc.alloc(&slots, 2 * kRepl * repl_stride(G)));
    FPH_TRY(sc.alloc(&arrived, kCtrs * kCtrStride));
    FPH_CUDA_TRY(cudaMemsetAsync(arrived, 0, sizeof(unsigned long long) * kCtrs * kCtrStride, stream));
    if (!use_smem) FPH_TRY(sc.alloc(&mind, n));
    // large resident clouds: the Morton-sorted variant (warps skip the
    // iterations that cannot change their points)
    static const bool sorted_on = [] {
        const char* e = getenv("FPH_FPS_SORTED");
        return !(e && e[0] == '0');
    }();
    static const long long sorted_min = [] {  // FPH_FPS_SORTED_MIN: tests force it on small clouds
        const char* e = getenv("FPH_FPS_SORTED_MIN");
        return e ? atoll(e) : (long long)kSortedMin;
    }();
    const int pt_need = (chunk + kResNT - 1) / kResNT;
    if (use_smem && sorted_on && n >= sorted_min && pt_need <= kSortedMaxPT && k > 1) {
        double *sx = nullptr, *sy = nullptr, *sz = nullptr;
        int *sidx = nullptr, *spos = nullptr;
        FPH_TRY(morton_sort(d_x, d_y, d_z, n, sc, stream, &sx, &sy, &sz, &sidx, &spos));
        int rc = FPH_OK;
#define FPH_SORTED_CASE(P)                                                                     \
    case P:                                                                                    \
        rc = launch_sorted<P>(d_x, d_y, d_z, sx, sy, sz, sidx, spos, n, k, start, chunk, G,   \
                              slots, arrived, d_out, stream);                                  \
        break;
        switch (pt_need) {
            FPH_SORTED_CASE(1)
            FPH_SORTED_CASE(2)
            FPH_SORTED_CASE(3)
            FPH_SORTED_CASE(4)
            FPH_SORTED_CASE(5)
            FPH_SORTED_CASE(6)
            FPH_SORTED_CASE(7)
            FPH_SORTED_CASE(8)
            FPH_SORTED_CASE(9)
            FPH_SORTED_CASE(10)
            FPH_SORTED_CASE(11)
            FPH_SORTED_CASE(12)
            FPH_SORTED_CASE(13)
            FPH_SORTED_CASE(14)
            default:
                FPH_SORTED_CASE(15)
        }
#undef FPH_SORTED_CASE
        if (rc != FPH_OK) return rc;
        FPH_CUDA_TRY(cudaGetLastError());
        return FPH_OK;
    }
    if (use_smem) {
        int rc = FPH_OK;
#define FPH_RESIDENT_CASE(P)                                                                   \
    case P:                                                                                    \
        rc = launch_resident<P>(d_x, d_y, d_z, n, k, start, chunk, G, slots, arrived, d_out,   \
                                stream);                                                       \
        break;
        static_assert(kResNT == 1024 || kResNT == 512, "resident kernel: 512 or 1024 threads");
        switch ((chunk + kResNT - 1) / kResNT) {
            FPH_RESIDENT_CASE(1)
            FPH_RESIDENT_CASE(2)
            FPH_RESIDENT_CASE(3)
            FPH_RESIDENT_CASE(4)
            FPH_RESIDENT_CASE(5)
            FPH_RESIDENT_CASE(6)
            FPH_RESIDENT_CASE(7)
            FPH_RESIDENT_CASE(8)
#if FPH_FPS_RES_NT <= 512
            FPH_RESIDENT_CASE(9)
            FPH_RESIDENT_CASE(10)
            FPH_RESIDENT_CASE(11)
            FPH_RESIDENT_CASE(12)
            FPH_RESIDENT_CASE(13)
            FPH_RESIDENT_CASE(14)
            FPH_RESIDENT_CASE(15)
            FPH_RESIDENT_CASE(16)
            FPH_RESIDENT_CASE(17)
            default:
                FPH_RESIDENT_CASE(18)
#else
            default:
                FPH_RESIDENT_CASE(9)
#endif
        }
#undef FPH_RESIDENT_CASE
        if (rc != FPH_OK) return rc;
    } else {
        void* args[] = {(void*)&d_x,   (void*)&d_y,  (void*)&d_z,   (void*)&n,
                        (void*)&k,     (void*)&start, (void*)&chunk, (void*)&mind,
                        (void*)&slots, (void*)&arrived, (void*)&d_out};
        FPH_CUDA_TRY(cudaLaunchCooperativeKernel((void*)fps_kernel, dim3(G), dim3(kFpsThreads),
                                                 args, 0, stream));
    }
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

}  // namespace fph

namespace fph {

int fps_batched(const double* d_x, const double* d_y, const double* d_z, int batch, int n, int k,
                int start, long long* d_out, cudaStream_t stream) {
    if (k < 1 || k > n || start < 0 || start >= n || batch < 0) {
        set_error("farthest point sampling: need 1 <= k <= n and 0 <= start < n");
        return FPH_EARG;
    }
    if (batch == 0) return FPH_OK;
    int dev = 0, sms = 0, max_smem = 0;
    FPH_CUDA_TRY(cudaGetDevice(&dev));
    FPH_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FPH_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const int cap = min(kFpsThreads * kFpsMaxPT, (max_smem - kStaticSmem) / (3 * (int)sizeof(double)));
    const int cpg = (n + cap - 1) / cap;
    if (cpg > sms || cpg > kMaxSlots) return FPH_EARG;  // caller falls back to one cloud at a time
    const int ngroups = min(sms / cpg, batch);
    const int chunk = (n + cpg - 1) / cpg;
    Scratch sc(stream);
    SlotXYZ* slots_xyz = nullptr;
    unsigned long long* arrived = nullptr;
    FPH_TRY(sc.alloc(&slots_xyz, 2 * cpg * ngroups));
    FPH_TRY(sc.alloc(&arrived, ngroups));
    Slot* slots = reinterpret_cast<Slot*>(slots_xyz);
    FPH_CUDA_TRY(cudaMemsetAsync(arrived, 0, sizeof(unsigned long long) * ngroups, stream));
    const int grid = ngroups * cpg;
    int rc = FPH_OK;
#define FPH_BATCHED_CASE(P)                                                                    \
    case P:                                                                                    \
        rc = launch_batched<P>(d_x, d_y, d_z, batch, n, k, start, cpg, chunk, grid, slots,     \
                               arrived, d_out, stream);                                        \
        break;
    switch ((chunk + kResNT - 1) / kResNT) {
        FPH_BATCHED_CASE(1)
        FPH_BATCHED_CASE(2)
        FPH_BATCHED_CASE(3)
        FPH_BATCHED_CASE(4)
        FPH_BATCHED_CASE(5)
        FPH_BATCHED_CASE(6)
        FPH_BATCHED_CASE(7)
        FPH_BATCHED_CASE(8)
#if FPH_FPS_RES_NT <= 512
        FPH_BATCHED_CASE(9)
        FPH_BATCHED_CASE(10)
        FPH_BATCHED_CASE(11)
        FPH_BATCHED_CASE(12)
        FPH_BATCHED_CASE(13)
        FPH_BATCHED_CASE(14)
        FPH_BATCHED_CASE(15)
        FPH_BATCHED_CASE(16)
        FPH_BATCHED_CASE(17)
        default:
            FPH_BATCHED_CASE(18)
#else
        default:
            FPH_BATCHED_CASE(9)
#endif
    }
#undef FPH_BATCHED_CASE
    if (rc != FPH_OK) return rc;
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

}  // namespace fph
