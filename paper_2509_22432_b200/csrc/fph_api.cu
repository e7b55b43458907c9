// fph_api.cu -- extern "C" entry points (include/floodph_b200.h).
//
// Host-memory calls stage inputs on the current device, run on a private
// stream and copy results back; device-memory calls run on the caller's
// stream.  Scratch comes from the stream-ordered allocator (cudaMallocAsync)
// whose pool is kept warm, so repeated calls do not pay cudaMalloc.
#include <array>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/floodph_b200.h"
#include "fph_flood.cuh"
#include "fph_grid.cuh"

#include <cub/cub.cuh>

namespace fph {

static thread_local char g_err[1024] = "";
static double g_occupancy = 2.0;
static double g_pairs_per_task = 0.0;
static bool g_profile = false;
static int g_algo = 1;
static int g_reps_target = 512;
static int g_team_threshold = 0;  // auto (derived per launch on the device)
static double g_exact_pairs = 65536.0;
static long long g_exact_cand[4] = {0, 0, 1000, 0};
#ifndef FPH_SPARSE_PPL
#define FPH_SPARSE_PPL 50.0
#endif
constexpr double kSparsePPL = FPH_SPARSE_PPL;
static thread_local long long g_launches = 0;

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void count_launches(int n) { g_launches += n; }

namespace {

__global__ void soa_kernel(const double* __restrict__ pts, long long n, int dim,
                           double* __restrict__ x, double* __restrict__ y,
                           double* __restrict__ z) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    x[i] = pts[i * dim];
    y[i] = pts[i * dim + 1];
    z[i] = dim == 3 ? pts[i * dim + 2] : 0.0;
}

__global__ void pad3_kernel(const double* __restrict__ pts, long long n, int dim,
                            double* __restrict__ out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i * 3] = pts[i * dim];
    out[i * 3 + 1] = pts[i * dim + 1];
    out[i * 3 + 2] = dim == 3 ? pts[i * dim + 2] : 0.0;
}

__global__ void pad4_kernel(const int* __restrict__ s, long long n, int k, int* __restrict__ out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int j = 0; j < 4; ++j) out[i * 4 + j] = j <= k ? s[i * (k + 1) + j] : -1;
}

// rows rank, rank + world, ... of an n x (k+1) table, padded to 4 ids
__global__ void pad4_shard_kernel(const int* __restrict__ s, long long n_out, int k, int rank,
                                  int world, int* __restrict__ out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_out) return;
    const long long row = rank + i * world;
    for (int j = 0; j < 4; ++j) out[i * 4 + j] = j <= k ? s[row * (k + 1) + j] : -1;
}

// 0-simplices i = 0..n-1 as (i, -1, -1, -1) rows
__global__ void vertex_ids_kernel(long long n, int* __restrict__ out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i * 4] = (int)i;
    out[i * 4 + 1] = out[i * 4 + 2] = out[i * 4 + 3] = -1;
}

// listed rows of an n_all x (k+1) table, padded to 4 ids (rows out of range
// give -1 ids and are rejected by the caller's validation upstream)
__global__ void pad4_rows_kernel(const int* __restrict__ s, long long n_all,
                                 const long long* __restrict__ rows, long long n_out, int k,
                                 int* __restrict__ out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n_out) return;
    const long long row = rows[i];
    const bool ok = row >= 0 && row < n_all;
    for (int j = 0; j < 4; ++j) out[i * 4 + j] = (ok && j <= k) ? s[row * (k + 1) + j] : -1;
}

__global__ void fill_kernel(double* out, long long n, double v) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) out[i] = v;
}

unsigned blocks_for(long long n) { return (unsigned)((n + 255) / 256); }

// Library streams, created once per device and kept: stream 0 (unused since
// host-memory calls moved to per-thread streams), streams 1 + 3 g + (k - 1)
// the dimension-k interior terms
// of a call holding grid slot g (run_interiors; higher dimensions at higher
// priority).
constexpr int kLibStreams = 1 + 3 * kGridSlots;
std::mutex g_stream_mu;
std::map<int, std::array<cudaStream_t, kLibStreams>> g_streams;

int lib_stream(int slot, cudaStream_t* out) {
    int dev = 0;
    FPH_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_stream_mu);
    auto it = g_streams.find(dev);
    if (it == g_streams.end()) {
        std::array<cudaStream_t, kLibStreams> st{};
        int lo = 0, hi = 0;
        FPH_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        for (int i = 0; i < kLibStreams; ++i)
            FPH_CUDA_TRY(cudaStreamCreateWithPriority(&st[i], cudaStreamNonBlocking,
                                                      i >= 1 && (i - 1) % 3 >= 1 ? hi : lo));
        it = g_streams.emplace(dev, st).first;
    }
    *out = it->second[slot];
    return FPH_OK;
}

// Host-memory calls run on a stream of the calling thread (one per thread
// and device, created on first use, kept): calls from different host
// threads overlap on the device -- the next call's copies and grid build
// under the current call's search -- while each call still returns only
// when its own work is done.
int thread_host_stream(cudaStream_t* out) {
    int dev = 0;
    FPH_CUDA_TRY(cudaGetDevice(&dev));
    thread_local std::map<int, cudaStream_t> streams;
    auto it = streams.find(dev);
    if (it == streams.end()) {
        cudaStream_t st = nullptr;
        FPH_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        it = streams.emplace(dev, st).first;
    }
    *out = it->second;
    return FPH_OK;
}

// Host-call context: the calling thread's library stream on the current
// device (host calls), or the caller's stream (device calls)
struct HostCtx {
    cudaStream_t stream = nullptr;
    int init(int memory, void* user_stream) {
        if (memory == FPH_MEM_DEVICE) {
            stream = static_cast<cudaStream_t>(user_stream);
            return FPH_OK;
        }
        return thread_host_stream(&stream);
    }
};

// The search kernels read the grid's parameters from a constant-memory slot
// (fph_search.cu c_grid; one copy of the kernels per slot, kGridSlots per
// device).  A call that launches them takes the next slot of its device
// round-robin and holds it from the copy of its grid into the slot until its
// kernels are queued; the next call on that slot waits (on the device) for
// an event recorded after them, so the GPU never rewrites a slot under
// running kernels.  Calls on different slots run concurrently.
struct DevSlots {
    std::mutex mu[kGridSlots];
    cudaEvent_t free_ev[kGridSlots] = {};
    unsigned long long ev_capture[kGridSlots] = {};  // capture id of the record (0: none)
    std::atomic<unsigned> next{0};
};
std::mutex g_slot_map_mu;
std::map<int, DevSlots*> g_slots;

struct GridSlot {
    DevSlots* ds = nullptr;
    int index = 0;
    cudaStream_t stream = nullptr;
    bool capturing = false;
    unsigned long long capture_id = 0;
    // cloud_bytes: the call's cloud (n x dim float64); clouds of at least
    // FPH_BIG_MIN_BYTES (default 64 MiB, i.e. beyond L2 once binned) take
    // the big-cloud build of the search kernels (kBigSlot)
    int acquire(const Grid* d_grid, cudaStream_t s, size_t cloud_bytes) {
        int dev = 0;
        FPH_CUDA_TRY(cudaGetDevice(&dev));
        {
            std::lock_guard<std::mutex> lock(g_slot_map_mu);
            auto it = g_slots.find(dev);
            if (it == g_slots.end()) it = g_slots.emplace(dev, new DevSlots).first;
            ds = it->second;
        }
        // Slots in use (FPH_GRID_SLOTS, default 1).  Two let the search
        // kernels of two calls overlap; measured on modelnet_batch (64 calls
        // on two streams) the graph replay gains 154 -> 144 ms but the eager
        // calls lose 143 -> 147 ms and host-memory calls 194 -> 215 ms: the
        // overlap that pays is a call's grid build and set-up under the
        // previous call's search, which one slot already allows.
        static const int nslots = [] {
            const char* e = getenv("FPH_GRID_SLOTS");
            const int v = e ? atoi(e) : 1;
            return v >= 1 && v <= 2 ? v : 1;
        }();
        static const size_t big_bytes = [] {
            const char* e = getenv("FPH_BIG_MIN_BYTES");
            return e ? (size_t)atoll(e) : ((size_t)64 << 20);
        }();
        index = cloud_bytes >= big_bytes ? kBigSlot
                                         : (int)(ds->next.fetch_add(1) % (unsigned)nslots);
        ds->mu[index].lock();
        stream = s;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        FPH_CUDA_TRY(cudaStreamGetCaptureInfo(s, &cs, &capture_id));
        capturing = cs != cudaStreamCaptureStatusNone;
        if (!capturing) capture_id = 0;
        // an event recorded in the same capture (a CUDA graph of a step) is
        // a dependency inside the graph; one recorded outside it cannot be
        // waited on there, and the graph's own order stands in for it
        if (ds->free_ev[index] && ds->ev_capture[index] == capture_id)
            FPH_CUDA_TRY(cudaStreamWaitEvent(s, ds->free_ev[index], 0));
        return set_search_grid(index, d_grid, s);
    }
    ~GridSlot() {
        if (!ds) return;
        if (!ds->free_ev[index])
            cudaEventCreateWithFlags(&ds->free_ev[index], cudaEventDisableTiming);
        if (ds->free_ev[index] && cudaEventRecord(ds->free_ev[index], stream) == cudaSuccess)
            ds->ev_capture[index] = capture_id;
        ds->mu[index].unlock();
    }
};

// a host-memory call returns once its stream is drained (on errors too)
int host_finish(const HostCtx& hc, int memory, int rc) {
    if (memory != FPH_MEM_HOST) return rc;
    const cudaError_t e = cudaStreamSynchronize(hc.stream);
    if (rc == FPH_OK && e != cudaSuccess) {
        set_error("cudaStreamSynchronize: %s", cudaGetErrorString(e));
        return FPH_ECUDA;
    }
    return rc;
}

// frees a GridStore on every exit path
struct GridGuard {
    GridStore& gs;
    cudaStream_t stream;
    ~GridGuard() { gs.free_all(stream); }
};

int ensure_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        set_error("no CUDA device available (%s)", e == cudaSuccess ? "0 devices"
                                                                   : cudaGetErrorString(e));
        return FPH_ECUDA;
    }
    static bool pool_ready = false;
    if (!pool_ready) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_ready = true;
    }
    return FPH_OK;
}

// Stage a host or device array as a device pointer.
template <class T>
int stage_in(Scratch& sc, const T* src, size_t count, int memory, const T** out) {
    if (memory == FPH_MEM_DEVICE || count == 0) {
        *out = src;
        return FPH_OK;
    }
    T* d = nullptr;
    FPH_TRY(sc.alloc(&d, count));
    FPH_CUDA_TRY(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, sc.stream));
    *out = d;
    return FPH_OK;
}

int check_cloud(const double* points, int64_t n, int32_t dim) {
    if (!points || n < 1) {
        set_error("point cloud needs at least one point");
        return FPH_EARG;
    }
    if (dim != 2 && dim != 3) {
        set_error("dimension must be 2 or 3, got %d", (int)dim);
        return FPH_EARG;
    }
    if (n > 0x7fffffffLL) {
        set_error("clouds above 2^31 points are not supported");
        return FPH_EARG;
    }
    return FPH_OK;
}

FloodTuning current_tuning(double points_per_landmark = 0.0, int grid_slot = 0) {
    FloodTuning t;
    t.points_per_landmark = points_per_landmark;
    t.pairs_per_task = g_pairs_per_task;
    t.profile = g_profile;
    t.algo = g_algo;
    t.reps_target = g_reps_target;
    t.team_threshold = g_team_threshold;
    t.exact_pairs = g_exact_pairs;
    static const double env_pairs = [] {  // experiments: FPH_EXACT_PAIRS overrides the default
        const char* e = getenv("FPH_EXACT_PAIRS");
        return e ? atof(e) : -1.0;
    }();
    if (env_pairs >= 0.0 && g_exact_pairs == 65536.0) t.exact_pairs = env_pairs;
    for (int i = 0; i < 4; ++i) t.exact_cand[i] = g_exact_cand[i];
    // sparse clouds (few points per landmark, e.g. configs[0]'s 20): the
    // one-pass exact phase A stays cheaper up to 2500 triangle candidates
    if (g_exact_cand[2] == 1000 && points_per_landmark > 0.0 && points_per_landmark < kSparsePPL)
        t.exact_cand[2] = 2500;
    t.grid_slot = grid_slot;
    return t;
}

// grid_build, timed with events when profiling is on (fph_flood_stats [23])
int build_grid_timed(const double* d_pts, int n, int dim, cudaStream_t stream, GridStore* gs,
                     bool keep_index = false) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (g_profile) {
        FPH_CUDA_TRY(cudaEventCreate(&a));
        FPH_CUDA_TRY(cudaEventCreate(&b));
        FPH_CUDA_TRY(cudaEventRecord(a, stream));
    }
    FPH_TRY(grid_build(d_pts, n, dim, 0.0, g_occupancy, stream, gs, keep_index));
    if (g_profile) {
        FPH_CUDA_TRY(cudaEventRecord(b, stream));
        profile_push_grid(a, b);
    }
    return FPH_OK;
}

int check_resolution(int m) {
    if (m < 1 || m > kMaxResolution) {
        set_error("grid_resolution must be in [1, %d], got %d", kMaxResolution, m);
        return FPH_EARG;
    }
    return FPH_OK;
}

}  // namespace
}  // namespace fph

using namespace fph;

extern "C" {

int fph_abi_version(void) { return FPH_ABI_VERSION; }

const char* fph_last_error(void) { return g_err; }

int fph_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int fph_set_tuning(double cell_occupancy, double pairs_per_task) {
    g_occupancy = cell_occupancy > 0 ? cell_occupancy : 2.0;
    g_pairs_per_task = pairs_per_task > 0 ? pairs_per_task : 0.0;
    return FPH_OK;
}

int fph_flood_complete(const double* interior_sq, const int32_t* facets, int64_t n, int32_t k,
                       const double* lower_sq, double* out_sq, void* stream) {
    g_err[0] = 0;
    if (k < 1 || k > 3 || n < 0) {
        set_error("fph_flood_complete: need 1 <= k <= 3 and n >= 0");
        return FPH_EARG;
    }
    FPH_TRY(ensure_device());
    count_launches(1);
    return flood_complete(interior_sq, facets, (int)n, k, lower_sq, out_sq,
                          static_cast<cudaStream_t>(stream));
}

int fph_set_search(int32_t algo, int32_t reps_target, int32_t team_threshold) {
    if (algo < 0 || algo > 1) {
        set_error("algo must be 0 (brute force) or 1 (bounded search)");
        return FPH_EARG;
    }
    g_algo = algo;
    g_reps_target = reps_target > 0 ? reps_target : 512;
    g_team_threshold = team_threshold;
    return FPH_OK;
}

int fph_set_exact_pairs(double pairs) {
    g_exact_pairs = pairs >= 0 ? pairs : 65536.0;
    return FPH_OK;
}

int fph_set_exact_candidates(int32_t k, int64_t candidates) {
    if (k < 0 || k > 3) {
        set_error("k must be in [0, 3]");
        return FPH_EARG;
    }
    g_exact_cand[k] = candidates > 0 ? candidates : 0;
    return FPH_OK;
}

int fph_set_profiling(int32_t on) {
    g_profile = on != 0;
    return FPH_OK;
}

int fph_flood_stats(double* out, int32_t reset) {
    g_err[0] = 0;
    FPH_TRY(ensure_device());
    return flood_stats(out, reset);
}

double fph_fp32_peak_tflops(void) {
    if (ensure_device() != FPH_OK) return 0.0;
    int dev = 0;
    cudaGetDevice(&dev);
    return ffma2_peak_tflops(dev);
}

double fph_tmem_min_rate(void) {
    if (ensure_device() != FPH_OK) return 0.0;
    int dev = 0;
    cudaGetDevice(&dev);
    return tmem_min_rate(dev);
}

double fph_tilemin_rate(void) {
    if (ensure_device() != FPH_OK) return 0.0;
    int dev = 0;
    cudaGetDevice(&dev);
    return tilemin_rate(dev);
}

int fph_debug_simplex_cycles(int32_t enable, int64_t* out, int64_t cap, int64_t* n) {
    g_err[0] = 0;
    if (n) {  // fetch first (waits for the device), then switch
        long long nn = 0;
        FPH_TRY(debug_fetch(reinterpret_cast<long long*>(out), out ? cap : 0, &nn));
        *n = nn;
    }
    debug_enable(enable != 0);
    return FPH_OK;
}

int64_t fph_launch_count(int32_t reset) {
    long long v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

int fph_farthest_point_sampling(const double* points, int64_t n, int32_t dim, int64_t k,
                                int64_t start, int64_t* out_indices, int32_t memory,
                                void* stream) {
    g_err[0] = 0;
    FPH_TRY(check_cloud(points, n, dim));
    if (k < 1 || k > n) {
        set_error("k must be in [1, %lld], got %lld", (long long)n, (long long)k);
        return FPH_EARG;
    }
    if (start < 0 || start >= n) {
        set_error("start must be in [0, %lld), got %lld", (long long)n, (long long)start);
        return FPH_EARG;
    }
    FPH_TRY(ensure_device());
    HostCtx hc;
    FPH_TRY(hc.init(memory, stream));
    // the body runs in a lambda so that every exit path below still waits for
    // the copies of a host-memory call (the caller may free its buffers)
    const int rc = [&]() -> int {
        int rc = FPH_OK;
        Scratch sc(hc.stream);
        const double* d_pts = nullptr;
        FPH_TRY(stage_in(sc, points, (size_t)n * dim, memory, &d_pts));
        double *x, *y, *z;
        FPH_TRY(sc.alloc(&x, n));
        FPH_TRY(sc.alloc(&y, n));
        FPH_TRY(sc.alloc(&z, n));
        soa_kernel<<<blocks_for(n), 256, 0, hc.stream>>>(d_pts, n, dim, x, y, z);
        count_launches(1);
        long long* d_out = reinterpret_cast<long long*>(out_indices);
        if (memory == FPH_MEM_HOST) FPH_TRY(sc.alloc(&d_out, k));
        rc = fps_run(x, y, z, (int)n, (int)k, (int)start, d_out, hc.stream);
        count_launches(1);
        if (rc == FPH_OK && memory == FPH_MEM_HOST) {
            FPH_CUDA_TRY(cudaMemcpyAsync(out_indices, d_out, sizeof(long long) * k,
                                         cudaMemcpyDeviceToHost, hc.stream));
        }
        return rc;
    }();
    return host_finish(hc, memory, rc);
}

int fph_farthest_point_sampling_batched(const double* points, int64_t batch, int64_t n,
                                        int32_t dim, int64_t k, int64_t start,
                                        int64_t* out_indices, int32_t memory, void* stream) {
    g_err[0] = 0;
    if (batch < 0) {
        set_error("batch must be nonnegative");
        return FPH_EARG;
    }
    if (batch == 0) return FPH_OK;
    FPH_TRY(check_cloud(points, n, dim));
    if (k < 1 || k > n) {
        set_error("k must be in [1, %lld], got %lld", (long long)n, (long long)k);
        return FPH_EARG;
    }
    if (start < 0 || start >= n) {
        set_error("start must be in [0, %lld), got %lld", (long long)n, (long long)start);
        return FPH_EARG;
    }
    if (batch * n > 0x7fffffffLL) {
        set_error("batch x n above 2^31 points is not supported");
        return FPH_EARG;
    }
    FPH_TRY(ensure_device());
    HostCtx hc;
    FPH_TRY(hc.init(memory, stream));
    // the body runs in a lambda so that every exit path below still waits for
    // the copies of a host-memory call (the caller may free its buffers)
    const int rc = [&]() -> int {
        int rc = FPH_OK;
        Scratch sc(hc.stream);
        const long long total = batch * n;
        const double* d_pts = nullptr;
        FPH_TRY(stage_in(sc, points, (size_t)total * dim, memory, &d_pts));
        double *x, *y, *z;
        FPH_TRY(sc.alloc(&x, total));
        FPH_TRY(sc.alloc(&y, total));
        FPH_TRY(sc.alloc(&z, total));
        soa_kernel<<<blocks_for(total), 256, 0, hc.stream>>>(d_pts, total, dim, x, y, z);
        count_launches(1);
        long long* d_out = reinterpret_cast<long long*>(out_indices);
        if (memory == FPH_MEM_HOST) FPH_TRY(sc.alloc(&d_out, (size_t)batch * k));
        rc = fps_batched(x, y, z, (int)batch, (int)n, (int)k, (int)start, d_out, hc.stream);
        count_launches(1);
        if (rc == FPH_EARG) {  // clouds too large to group: one at a time
            rc = FPH_OK;
            for (int64_t b = 0; b < batch && rc == FPH_OK; ++b) {
                rc = fps_run(x + b * n, y + b * n, z + b * n, (int)n, (int)k, (int)start,
                             d_out + b * k, hc.stream);
                count_launches(1);
            }
        }
        if (rc == FPH_OK && memory == FPH_MEM_HOST)
            FPH_CUDA_TRY(cudaMemcpyAsync(out_indices, d_out, sizeof(long long) * batch * k,
                                         cudaMemcpyDeviceToHost, hc.stream));
        return rc;
    }();
    return host_finish(hc, memory, rc);
}

int fph_flood_interior(const double* points, int64_t n_points, int32_t dim,
                       const double* landmarks, int64_t n_landmarks, const int32_t* simplices,
                       int64_t n_simplices, int32_t k, int32_t grid_resolution,
                       int32_t subset_mode, double* out_sq, int32_t memory, void* stream) {
    g_err[0] = 0;
    FPH_TRY(check_cloud(points, n_points, dim));
    FPH_TRY(check_resolution(grid_resolution));
    if (k < 0 || k > 3 || n_landmarks < 1) {
        set_error("need 0 <= k <= 3 and landmarks");
        return FPH_EARG;
    }
    if (n_simplices == 0) return FPH_OK;
    FPH_TRY(ensure_device());
    HostCtx hc;
    FPH_TRY(hc.init(memory, stream));
    // the body runs in a lambda so that every exit path below still waits for
    // the copies of a host-memory call (the caller may free its buffers)
    const int rc = [&]() -> int {
        int rc = FPH_OK;
        Scratch sc(hc.stream);
        const double *d_pts, *d_lm;
        const int32_t* d_s;
        FPH_TRY(stage_in(sc, points, (size_t)n_points * dim, memory, &d_pts));
        FPH_TRY(stage_in(sc, landmarks, (size_t)n_landmarks * dim, memory, &d_lm));
        FPH_TRY(stage_in(sc, simplices, (size_t)n_simplices * 4, memory, &d_s));
        double* lm3;
        FPH_TRY(sc.alloc(&lm3, (size_t)n_landmarks * 3));
        pad3_kernel<<<blocks_for(n_landmarks), 256, 0, hc.stream>>>(d_lm, n_landmarks, dim, lm3);
        count_launches(1);
        GridStore gs;
        GridGuard gg{gs, hc.stream};
        FPH_TRY(build_grid_timed(d_pts, (int)n_points, dim, hc.stream, &gs));
        count_launches(4);
        double* d_out = out_sq;
        if (memory == FPH_MEM_HOST) FPH_TRY(sc.alloc(&d_out, n_simplices));
        GridSlot slot;
        FPH_TRY(slot.acquire(gs.d_grid, hc.stream, (size_t)n_points * dim * sizeof(double)));
        rc = flood_interior(gs.d_grid, lm3, d_s, (int)n_simplices, k, grid_resolution, subset_mode,
                            d_out, current_tuning((double)n_points / n_landmarks, slot.index),
                            hc.stream);
        count_launches(4);
        if (rc == FPH_OK && memory == FPH_MEM_HOST)
            FPH_CUDA_TRY(cudaMemcpyAsync(out_sq, d_out, sizeof(double) * n_simplices,
                                         cudaMemcpyDeviceToHost, hc.stream));
        return rc;
    }();
    return host_finish(hc, memory, rc);
}

int fph_flood_samples(const double* points, int64_t n_points, int32_t dim,
                      const double* landmarks, int64_t n_landmarks, const int32_t* simplices,
                      int64_t n_simplices, int32_t k, const double* samples, int32_t n_samples,
                      int32_t subset_mode, double* out_sq, int32_t memory, void* stream) {
    g_err[0] = 0;
    FPH_TRY(check_cloud(points, n_points, dim));
    if (k < 0 || k > 3 || n_samples < 1 || n_landmarks < 1) {
        set_error("need 0 <= k <= 3, n_samples >= 1 and landmarks");
        return FPH_EARG;
    }
    if (n_simplices == 0) return FPH_OK;
    FPH_TRY(ensure_device());
    HostCtx hc;
    FPH_TRY(hc.init(memory, stream));
    // the body runs in a lambda so that every exit path below still waits for
    // the copies of a host-memory call (the caller may free its buffers)
    const int rc = [&]() -> int {
        int rc = FPH_OK;
        Scratch sc(hc.stream);
        const double *d_pts, *d_lm, *d_smp;
        const int32_t* d_s;
        FPH_TRY(stage_in(sc, points, (size_t)n_points * dim, memory, &d_pts));
        FPH_TRY(stage_in(sc, landmarks, (size_t)n_landmarks * dim, memory, &d_lm));
        FPH_TRY(stage_in(sc, simplices, (size_t)n_simplices * 4, memory, &d_s));
        const long long nrow = (long long)n_simplices * n_samples;
        FPH_TRY(stage_in(sc, samples, (size_t)nrow * dim, memory, &d_smp));
        double *lm3, *smp3;
        FPH_TRY(sc.alloc(&lm3, (size_t)n_landmarks * 3));
        FPH_TRY(sc.alloc(&smp3, (size_t)nrow * 3));
        pad3_kernel<<<blocks_for(n_landmarks), 256, 0, hc.stream>>>(d_lm, n_landmarks, dim, lm3);
        pad3_kernel<<<blocks_for(nrow), 256, 0, hc.stream>>>(d_smp, nrow, dim, smp3);
        count_launches(2);
        GridStore gs;
        GridGuard gg{gs, hc.stream};
        FPH_TRY(build_grid_timed(d_pts, (int)n_points, dim, hc.stream, &gs));
        count_launches(4);
        double* d_out = out_sq;
        if (memory == FPH_MEM_HOST) FPH_TRY(sc.alloc(&d_out, n_simplices));
        GridSlot slot;
        FPH_TRY(slot.acquire(gs.d_grid, hc.stream, (size_t)n_points * dim * sizeof(double)));
        rc = flood_interior(gs.d_grid, lm3, d_s, (int)n_simplices, k, 1, subset_mode, d_out,
                            current_tuning((double)n_points / n_landmarks, slot.index), hc.stream, smp3,
                            n_samples);
        count_launches(4);
        if (rc == FPH_OK && memory == FPH_MEM_HOST)
            FPH_CUDA_TRY(cudaMemcpyAsync(out_sq, d_out, sizeof(double) * n_simplices,
                                         cudaMemcpyDeviceToHost, hc.stream));
        return rc;
    }();
    return host_finish(hc, memory, rc);
}

// Interior terms of dimensions 1..max_dim, concurrently on side streams
// forked from (and joined back into) `stream`.  With profiling on, the
// flooding time recorded is the fork-to-join interval.
static int run_interiors(const Grid* g, const double* lm3, int* const* s4, double* const* interior,
                         const int64_t* counts, int max_dim, int grid_resolution, int subset_mode,
                         FloodTuning tune, cudaStream_t stream) {
    cudaEvent_t fork = nullptr, done[4] = {nullptr, nullptr, nullptr, nullptr}, p0 = nullptr,
                p1 = nullptr;
    const bool prof = tune.profile;
    tune.profile = false;
    if (prof) {
        FPH_CUDA_TRY(cudaEventCreate(&p0));
        FPH_CUDA_TRY(cudaEventCreate(&p1));
        FPH_CUDA_TRY(cudaEventRecord(p0, stream));
    }
    FPH_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    FPH_CUDA_TRY(cudaEventRecord(fork, stream));
    int rc = FPH_OK;
    for (int k = 1; k <= max_dim && rc == FPH_OK; ++k) {
        if (counts[k] == 0) continue;
        // higher dimensions carry the longest chains: their CTAs are placed
        // first (higher stream priority), lower dimensions fill the tails
        cudaStream_t sk = nullptr;
        FPH_TRY(lib_stream(1 + 3 * tune.grid_slot + (k - 1), &sk));
        FPH_CUDA_TRY(cudaStreamWaitEvent(sk, fork, 0));
        rc = flood_interior(g, lm3, s4[k], (int)counts[k], k, grid_resolution, subset_mode,
                            interior[k], tune, sk);
        count_launches(4);
        FPH_CUDA_TRY(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
        FPH_CUDA_TRY(cudaEventRecord(done[k], sk));
    }
    for (int k = 1; k <= max_dim; ++k)
        if (done[k]) {
            FPH_CUDA_TRY(cudaStreamWaitEvent(stream, done[k], 0));
            cudaEventDestroy(done[k]);
        }
    cudaEventDestroy(fork);
    if (prof) {
        FPH_CUDA_TRY(cudaEventRecord(p1, stream));
        profile_push(p0, p1);
    }
    return rc;
}

// Interior terms of a subset of every dimension's simplices with one grid
// build: rows[k] (n_rows[k] indices) or, when rows is null, the interleaved
// share rank, rank + world, ...
static int flood_rows(const double* points, int64_t n_points, int32_t dim,
                      const double* landmarks, int64_t n_landmarks, int32_t max_dim,
                      const int64_t* counts, const int32_t* const* simplices,
                      const int64_t* const* rows, const int64_t* n_rows, int32_t rank,
                      int32_t world, int32_t grid_resolution, int32_t subset_mode,
                      double* const* out_interior, int32_t memory, void* stream) {
    g_err[0] = 0;
    FPH_TRY(check_cloud(points, n_points, dim));
    FPH_TRY(check_resolution(grid_resolution));
    if (max_dim < 1 || max_dim > 3 || n_landmarks < 1 || !counts || world < 1 || rank < 0 ||
        rank >= world) {
        set_error("need 1 <= max_dim <= 3, landmarks and 0 <= rank < world");
        return FPH_EARG;
    }
    FPH_TRY(ensure_device());
    HostCtx hc;
    FPH_TRY(hc.init(memory, stream));
    // the body runs in a lambda so that every exit path below still waits for
    // the copies of a host-memory call (the caller may free its buffers)
    const int rc = [&]() -> int {
        int rc = FPH_OK;
        Scratch sc(hc.stream);
        const double *d_pts, *d_lm;
        FPH_TRY(stage_in(sc, points, (size_t)n_points * dim, memory, &d_pts));
        FPH_TRY(stage_in(sc, landmarks, (size_t)n_landmarks * dim, memory, &d_lm));
        double* lm3;
        FPH_TRY(sc.alloc(&lm3, (size_t)n_landmarks * 3));
        pad3_kernel<<<blocks_for(n_landmarks), 256, 0, hc.stream>>>(d_lm, n_landmarks, dim, lm3);
        count_launches(1);
        GridStore gs;
        GridGuard gg{gs, hc.stream};
        FPH_TRY(build_grid_timed(d_pts, (int)n_points, dim, hc.stream, &gs));
        count_launches(4);
        FloodTuning tune = current_tuning((double)n_points / n_landmarks);
        int64_t mine[4] = {0, 0, 0, 0};
        int* s4[4] = {nullptr, nullptr, nullptr, nullptr};
        double* d_out[4] = {nullptr, nullptr, nullptr, nullptr};
        for (int k = 1; k <= max_dim && rc == FPH_OK; ++k) {
            const long long nk = counts[k];
            mine[k] = rows ? n_rows[k] : (nk > rank ? (nk - 1 - rank) / world + 1 : 0);
            if (mine[k] == 0) continue;
            const int32_t* d_s;
            FPH_TRY(stage_in(sc, simplices[k], (size_t)nk * (k + 1), memory, &d_s));
            FPH_TRY(sc.alloc(&s4[k], (size_t)mine[k] * 4));
            if (rows) {
                const int64_t* d_rows;
                FPH_TRY(stage_in(sc, rows[k], (size_t)mine[k], memory, &d_rows));
                pad4_rows_kernel<<<blocks_for(mine[k]), 256, 0, hc.stream>>>(
                    d_s, nk, reinterpret_cast<const long long*>(d_rows), mine[k], k, s4[k]);
            } else {
                pad4_shard_kernel<<<blocks_for(mine[k]), 256, 0, hc.stream>>>(d_s, mine[k], k, rank,
                                                                             world, s4[k]);
            }
            count_launches(1);
            d_out[k] = out_interior[k];
            if (memory == FPH_MEM_HOST) FPH_TRY(sc.alloc(&d_out[k], (size_t)mine[k]));
        }
        // every dimension's share concurrently, as in fph_flood_filtration
        GridSlot slot;
        if (rc == FPH_OK) rc = slot.acquire(gs.d_grid, hc.stream, (size_t)n_points * dim * sizeof(double));
        tune.grid_slot = slot.index;
        if (rc == FPH_OK) rc = run_interiors(gs.d_grid, lm3, s4, d_out, mine, max_dim,
                                            grid_resolution, subset_mode, tune, hc.stream);
        for (int k = 1; k <= max_dim && rc == FPH_OK; ++k)
            if (mine[k] > 0 && memory == FPH_MEM_HOST)
                FPH_CUDA_TRY(cudaMemcpyAsync(out_interior[k], d_out[k], sizeof(double) * mine[k],
                                             cudaMemcpyDeviceToHost, hc.stream));
        return rc;
    }();
    return host_finish(hc, memory, rc);
}

int fph_flood_shard(const double* points, int64_t n_points, int32_t dim,
                    const double* landmarks, int64_t n_landmarks, int32_t max_dim,
                    const int64_t* counts, const int32_t* const* simplices, int32_t rank,
                    int32_t world, int32_t grid_resolution, int32_t subset_mode,
                    double* const* out_interior, int32_t memory, void* stream) {
    return flood_rows(points, n_points, dim, landmarks, n_landmarks, max_dim, counts, simplices,
                      nullptr, nullptr, rank, world, grid_resolution, subset_mode, out_interior,
                      memory, stream);
}

int fph_flood_subset(const double* points, int64_t n_points, int32_t dim,
                     const double* landmarks, int64_t n_landmarks, int32_t max_dim,
                     const int64_t* counts, const int32_t* const* simplices,
                     const int64_t* const* rows, const int64_t* n_rows, int32_t grid_resolution,
                     int32_t subset_mode, double* const* out_interior, int32_t memory,
                     void* stream) {
    if (!rows || !n_rows) {
        g_err[0] = 0;
        set_error("fph_flood_subset: rows and n_rows are required");
        return FPH_EARG;
    }
    for (int k = 1; k <= max_dim && k <= 3; ++k)
        if (n_rows[k] < 0 || (n_rows[k] > 0 && !rows[k])) {
            set_error("fph_flood_subset: bad row list for dimension %d", k);
            return FPH_EARG;
        }
    return flood_rows(points, n_points, dim, landmarks, n_landmarks, max_dim, counts, simplices,
                      rows, n_rows, 0, 1, grid_resolution, subset_mode, out_interior, memory,
                      stream);
}

int fph_flood_filtration(const double* points, int64_t n_points, int32_t dim,
                         const double* landmarks, int64_t n_landmarks, int32_t max_dim,
                         const int64_t* counts, const int32_t* const* simplices,
                         const int32_t* const* facets, int32_t grid_resolution,
                         int32_t subset_mode, double* const* out_sq, int32_t memory,
                         void* stream) {
    g_err[0] = 0;
    FPH_TRY(check_cloud(points, n_points, dim));
    FPH_TRY(check_resolution(grid_resolution));
    if (max_dim < 0 || max_dim > 3 || n_landmarks < 1 || !counts) {
        set_error("need 0 <= max_dim <= 3 and landmarks");
        return FPH_EARG;
    }
    FPH_TRY(ensure_device());
    HostCtx hc;
    FPH_TRY(hc.init(memory, stream));
    // the body runs in a lambda so that every exit path below still waits for
    // the copies of a host-memory call (the caller may free its buffers)
    const int rc = [&]() -> int {
        int rc = FPH_OK;
        Scratch sc(hc.stream);
        const double *d_pts, *d_lm;
        FPH_TRY(stage_in(sc, points, (size_t)n_points * dim, memory, &d_pts));
        FPH_TRY(stage_in(sc, landmarks, (size_t)n_landmarks * dim, memory, &d_lm));
        double* lm3;
        FPH_TRY(sc.alloc(&lm3, (size_t)n_landmarks * 3));
        pad3_kernel<<<blocks_for(n_landmarks), 256, 0, hc.stream>>>(d_lm, n_landmarks, dim, lm3);
        count_launches(1);
        GridStore gs;
        GridGuard gg{gs, hc.stream};
        FPH_TRY(build_grid_timed(d_pts, (int)n_points, dim, hc.stream, &gs));
        count_launches(4);
        GridSlot slot;
        FPH_TRY(slot.acquire(gs.d_grid, hc.stream, (size_t)n_points * dim * sizeof(double)));
        const FloodTuning tune = current_tuning((double)n_points / n_landmarks, slot.index);
        double* d_vals[4] = {nullptr, nullptr, nullptr, nullptr};
        const int32_t* d_f[4] = {nullptr, nullptr, nullptr, nullptr};
        int* s4[4] = {nullptr, nullptr, nullptr, nullptr};
        double* interior[4] = {nullptr, nullptr, nullptr, nullptr};
        for (int k = 0; k <= max_dim && rc == FPH_OK; ++k) {
            const long long nk = counts[k];
            double* d_out = out_sq[k];
            if (memory == FPH_MEM_HOST) FPH_TRY(sc.alloc(&d_out, nk > 0 ? nk : 1));
            d_vals[k] = d_out;
            if (nk == 0) continue;
            if (k == 0) {
                if (subset_mode) {
                    fill_kernel<<<blocks_for(nk), 256, 0, hc.stream>>>(d_out, nk, 0.0);
                    count_launches(1);
                } else {
                    // vertices: nearest cloud point of each landmark
                    int* v4;
                    FPH_TRY(sc.alloc(&v4, (size_t)nk * 4));
                    vertex_ids_kernel<<<blocks_for(nk), 256, 0, hc.stream>>>(nk, v4);
                    count_launches(1);
                    rc = flood_interior(gs.d_grid, lm3, v4, (int)nk, 0, grid_resolution, 0, d_out,
                                        tune, hc.stream);
                    count_launches(4);
                }
                continue;
            }
            const int32_t* d_s;
            FPH_TRY(stage_in(sc, simplices[k], (size_t)nk * (k + 1), memory, &d_s));
            FPH_TRY(stage_in(sc, facets[k], (size_t)nk * (k + 1), memory, &d_f[k]));
            FPH_TRY(sc.alloc(&s4[k], (size_t)nk * 4));
            FPH_TRY(sc.alloc(&interior[k], (size_t)nk));
            pad4_kernel<<<blocks_for(nk), 256, 0, hc.stream>>>(d_s, nk, k, s4[k]);
            count_launches(1);
        }
        // The interior terms of the dimensions >= 1 are independent: each runs
        // on its own stream so one dimension's kernels fill the other's tail;
        // the facet completion then runs in increasing dimension.
        if (rc == FPH_OK) rc = run_interiors(gs.d_grid, lm3, s4, interior, counts, max_dim,
                                            grid_resolution, subset_mode, tune, hc.stream);
        for (int k = 1; k <= max_dim && rc == FPH_OK; ++k) {
            if (counts[k] == 0) continue;
            rc = flood_complete(interior[k], d_f[k], (int)counts[k], k, d_vals[k - 1], d_vals[k],
                                hc.stream);
            count_launches(1);
        }
        if (rc == FPH_OK && memory == FPH_MEM_HOST) {
            for (int k = 0; k <= max_dim; ++k)
                if (counts[k] > 0)
                    FPH_CUDA_TRY(cudaMemcpyAsync(out_sq[k], d_vals[k], sizeof(double) * counts[k],
                                                 cudaMemcpyDeviceToHost, hc.stream));
        }
        return rc;
    }();
    return host_finish(hc, memory, rc);
}

int fph_candidate_mask(const double* points, int64_t n_points, int32_t dim,
                       const double* landmarks, int64_t n_landmarks, const int32_t* cells,
                       int64_t n_cells, int32_t k, int64_t* out_offsets, int32_t* out_indices,
                       int64_t capacity) {
    g_err[0] = 0;
    FPH_TRY(check_cloud(points, n_points, dim));
    if (k < 0 || k > 3 || n_landmarks < 1 || n_cells < 0 || !out_offsets) {
        set_error("need 0 <= k <= 3, landmarks, n_cells >= 0 and out_offsets");
        return FPH_EARG;
    }
    out_offsets[0] = 0;
    if (n_cells == 0) return FPH_OK;
    FPH_TRY(ensure_device());
    HostCtx hc;
    FPH_TRY(hc.init(FPH_MEM_HOST, nullptr));
    const int rc = [&]() -> int {
        Scratch sc(hc.stream);
        const double *d_pts, *d_lm;
        const int32_t* d_c;
        FPH_TRY(stage_in(sc, points, (size_t)n_points * dim, FPH_MEM_HOST, &d_pts));
        FPH_TRY(stage_in(sc, landmarks, (size_t)n_landmarks * dim, FPH_MEM_HOST, &d_lm));
        FPH_TRY(stage_in(sc, cells, (size_t)n_cells * (k + 1), FPH_MEM_HOST, &d_c));
        double* lm3;
        int* c4;
        long long* d_off;
        FPH_TRY(sc.alloc(&lm3, (size_t)n_landmarks * 3));
        FPH_TRY(sc.alloc(&c4, (size_t)n_cells * 4));
        FPH_TRY(sc.alloc(&d_off, (size_t)n_cells + 1));
        pad3_kernel<<<blocks_for(n_landmarks), 256, 0, hc.stream>>>(d_lm, n_landmarks, dim, lm3);
        pad4_kernel<<<blocks_for(n_cells), 256, 0, hc.stream>>>(d_c, n_cells, k, c4);
        count_launches(2);
        GridStore gs;
        GridGuard gg{gs, hc.stream};
        FPH_TRY(grid_build(d_pts, (int)n_points, dim, 0.0, g_occupancy, hc.stream, &gs, true));
        FPH_CUDA_TRY(cudaMemsetAsync(d_off, 0, sizeof(long long), hc.stream));
        FPH_TRY(candidate_counts(gs.d_grid, lm3, c4, (int)n_cells, k, d_off + 1, hc.stream));
        size_t tb = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tb, d_off + 1, d_off + 1, (int)n_cells, hc.stream);
        unsigned char* tmp;
        FPH_TRY(sc.alloc(&tmp, tb));
        FPH_CUDA_TRY(cub::DeviceScan::InclusiveSum(tmp, tb, d_off + 1, d_off + 1, (int)n_cells,
                                                   hc.stream));
        FPH_CUDA_TRY(cudaMemcpyAsync(out_offsets, d_off, sizeof(long long) * (n_cells + 1),
                                     cudaMemcpyDeviceToHost, hc.stream));
        FPH_CUDA_TRY(cudaStreamSynchronize(hc.stream));
        const long long total = out_offsets[n_cells];
        if (!out_indices || total > capacity) return FPH_OK;  // sizes only
        if (total > 0x7fffffffLL) {
            set_error("candidate masks above 2^31 indices in one call are not supported");
            return FPH_EARG;
        }
        int* d_idx;
        FPH_TRY(sc.alloc(&d_idx, (size_t)total));
        FPH_TRY(candidate_fill(gs.d_grid, lm3, c4, (int)n_cells, k, d_off, total, d_idx, hc.stream));
        count_launches(3);
        FPH_CUDA_TRY(cudaMemcpyAsync(out_indices, d_idx, sizeof(int) * total,
                                     cudaMemcpyDeviceToHost, hc.stream));
        return FPH_OK;
    }();
    return host_finish(hc, FPH_MEM_HOST, rc);
}

}  // extern "C"
