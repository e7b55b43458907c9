// fph_flood.cuh -- flooding kernel interface (see fph_flood.cu).
#pragma once

#include "fph_common.cuh"

namespace fph {

struct SimplexGeom {
    double cx, cy, cz;  // Ritter center (float64, reference-exact)
    double r;           // Ritter radius
    double rho;         // candidate radius (sqrt(2) r, Lemma 4.2); 0 when unpruned
    Box box;            // candidate cell box
    int npc;            // point chunks (brute force)
    int nrp;            // row parts (brute force candidate splits)
};

// Largest grid resolution: template rows hold the compositions as ushort4.
constexpr int kMaxResolution = 65535;

struct FloodArgs {
    const Grid* gp;           // grid parameters (device memory, fph_grid.cu)
    const double* landmarks;  // n_landmarks x 3 (z = 0 for planar clouds)
    const int* simplices;     // n x 4, vertex ids, unused slots -1
    int n, k, m, P;
    int subset;               // landmarks are cloud points: Lemma 4.2 pruning
    int chunk_pts;            // brute force: points per task chunk = 256 * PPT
    double pairs_per_task;    // brute force: fp32 pairs per task
    const ushort4* tmpl;      // interior compositions, P rows (block-ordered)
    float* perpoint;          // n x P fp32 minima
    float* lower;             // per simplex: phase B's lower bound L (B | C kernels)
    double* out_sq;           // n squared interior maxima (-1: no interior row)
    // bounded search (algo 1): point blocks of <= 32 rows, reps
    const int* blk_off;       // nblk + 1 offsets into tmpl
    int nblk;
    int reps_target;          // candidates per representative pass
    int wt_off;               // byte offset of the (m + 1)-entry weight table in dynamic smem
    int* cand_count;          // per simplex: candidates in the Lemma-4.2 ball rows
    unsigned long long* stats;  // work counters (fph_flood_stats)
    int team_threshold;       // candidates above which a whole CTA takes the simplex
                              // (<= 0: derived on the device, see launch_search)
    const long long* team_thr_dev;  // that derived threshold (nullptr: use team_threshold)
    const double* explicit_pts;  // n x P x 3 sample rows (uniform-random sampler), or null
    long long* dbg;           // optional: per simplex 8 values (phase cycles, counters)
    double exact_pairs;       // bounded search: one exact pass when rows x candidates <= this
    long long exact_cand[4];  // bounded search: exact pass when candidates <= this, per dim
    double points_per_landmark;  // work estimate of a launch: n x P x this
};

// debug capture of flood_interior calls (per-simplex phase cycles, times):
// per simplex [cycles A, B, C, F; blocks; candidates; staged; team size;
// globaltimer start, end of A, B, C, F]
constexpr int kDbgFields = 16;
void debug_enable(bool on);
int debug_fetch(long long* out, long long cap, long long* n);

// algorithm 1 (fph_search.cu): warp-per-simplex bounded search.  Queued in
// two steps so a caller can put every dimension's set-up (team threshold,
// schedule sort) on the GPU before any dimension's persistent search kernels
// take the SMs: search_prepare, then search_run.
using SearchKernelFn = void (*)(const FloodArgs, const SimplexGeom*, const int*, int*, int*, int);
struct SearchPlan {
    FloodArgs b{};
    const SimplexGeom* d_geom = nullptr;
    cudaStream_t stream = nullptr;
    SearchKernelFn kern[4] = {nullptr, nullptr, nullptr, nullptr};
    int nk = 0, blocks = 0, smem = 0;
    float* d_lower = nullptr;
    long long* d_thr = nullptr;
    int *d_keys = nullptr, *d_order = nullptr, *d_iota = nullptr, *d_key_in = nullptr;
    int *d_counters = nullptr, *d_stage = nullptr;
    void* tmp = nullptr;
};
//
// fph_search.cu is compiled once per grid slot (FPH_GRID_SLOT 0, 1): each
// copy's kernels read their own __constant__ grid, so two calls holding
// different slots run concurrently on one device (a batch of clouds on two
// streams).  The copies' entry points live in namespaces slot0 / slot1.
// A third copy, slot2, is built for clouds too large for L2 (kBigSlot): 4
// search CTAs per SM (64 registers, 128-candidate tiles, rows' values in
// shared memory up to 256 rows), so more warps hide the DRAM latency of
// the candidate loads (box_10m 12.5 -> 10.75 ms; 3 CTAs: 11.2, 5: 11.1;
// on L2-resident clouds such builds lose 9-28% to spills and small tiles).
constexpr int kGridSlots = 3;
constexpr int kBigSlot = 2;
#define FPH_SEARCH_API                                                                     \
    int search_prepare(const FloodArgs& a, const SimplexGeom* d_geom, const int* d_cand,   \
                       cudaStream_t stream, SearchPlan* plan);                             \
    int search_run(SearchPlan& plan, bool release);                                        \
    int search_release(SearchPlan& plan);                                                  \
    int launch_search(const FloodArgs& a, const SimplexGeom* d_geom, const int* d_cand,    \
                      cudaStream_t stream);                                                \
    /* copy a device grid's parameters into this copy's constant slot, ordered on      */ \
    /* `stream` (the caller holds the slot, fph_api.cu GridSlot)                        */ \
    int set_search_grid(const Grid* d_grid, cudaStream_t stream);                          \
    /* dynamic shared memory of the search kernel for P rows at resolution m, and the  */ \
    /* device limit it must fit                                                         */ \
    size_t search_smem_bytes(int P, int m);                                                \
    size_t search_smem_limit();
namespace slot0 {
FPH_SEARCH_API
}
namespace slot1 {
FPH_SEARCH_API
}
namespace slot2 {
FPH_SEARCH_API
}
#undef FPH_SEARCH_API
inline int set_search_grid(int slot, const Grid* d_grid, cudaStream_t stream) {
    return slot == 2   ? slot2::set_search_grid(d_grid, stream)
           : slot == 1 ? slot1::set_search_grid(d_grid, stream)
                       : slot0::set_search_grid(d_grid, stream);
}

struct FloodTuning {
    int grid_slot = 0;            // the constant grid slot the caller holds (fph_api.cu GridSlot)
    double points_per_landmark = 0.0;  // cloud points / landmarks: scales the work estimate
    double pairs_per_task = 0.0;  // <= 0: default 2^21
    bool profile = false;         // time pass kernels with events
    int algo = 1;                 // 0: brute force over the Lemma-4.2 ball, 1: block search
    int reps_target = 384;        // block search: candidates per representative pass
    int team_threshold = 0;  // bounded search: CTA-cooperative simplices above this (<= 0: auto)
    double exact_pairs = 0.0;     // bounded search: exact pass below this many pairs
    long long exact_cand[4] = {0, 0, 0, 0};  // ... or below this many candidates (per dim)
};

// out[0..5]: work counters (see g_stats), out[6]: pass-kernel ms
int flood_stats(double* out, int reset);
void profile_push(cudaEvent_t a, cudaEvent_t b);
void profile_push_grid(cudaEvent_t a, cudaEvent_t b);
double ffma2_peak_tflops(int device);
// elements/s of tcgen05.ld + min over all SMs; pairs/s of the FFMA2 tile-min loop
double tmem_min_rate(int device);
double tilemin_rate(int device);

int choose_ppt(int P);

// The same in two steps: prepare queues the allocations, the setup kernel
// and the schedule sort; run queues the flooding kernels and frees.  (Queuing
// every dimension's set-up first, and all dimensions' kernels as one PDL chain
// on one stream, were both measured: no gain over concurrent per-dimension
// streams, docs/experiments.md.)
struct FloodJob;
int flood_interior_prepare(const Grid* d_grid, const double* d_landmarks3, const int* d_simplices,
                           int n, int k, int m, int subset, double* d_out_sq,
                           const FloodTuning& tune, cudaStream_t stream, FloodJob** job,
                           const double* d_explicit = nullptr, int explicit_rows = 0);
int flood_interior_run(FloodJob* job);

// Squared flood value over the relative-interior grid rows of every
// simplex (k = 0: the vertex itself), exactly as the reference computes it.
int flood_interior(const Grid* d_grid, const double* d_landmarks3, const int* d_simplices, int n,
                   int k, int m, int subset, double* d_out_sq, const FloodTuning& tune,
                   cudaStream_t stream, const double* d_explicit = nullptr, int explicit_rows = 0);

// out[i] = max(interior[i], lower[facets[i][j]] for j <= k)
int flood_complete(const double* d_interior, const int* d_facets, int n, int k,
                   const double* d_lower, double* d_out, cudaStream_t stream);

int fps_run(const double* d_x, const double* d_y, const double* d_z, int n, int k, int start,
            long long* d_out, cudaStream_t stream);

// `batch` equal clouds (SoA, cloud-major); FPH_EARG if one cloud needs more
// CTAs than there are SMs (the caller then runs fps_run per cloud)
int fps_batched(const double* d_x, const double* d_y, const double* d_z, int batch, int n, int k,
                int start, long long* d_out, cudaStream_t stream);

// candidate masks (fph_mask.cu): per simplex, the count / the ascending cloud
// indices of the points in its masking ball (needs a grid with idx)
int candidate_counts(const Grid* d_grid, const double* d_lm3, const int* d_cells4, int n, int k,
                     long long* d_counts, cudaStream_t stream);
int candidate_fill(const Grid* d_grid, const double* d_lm3, const int* d_cells4, int n, int k,
                   const long long* d_offsets, long long total, int* d_idx, cudaStream_t stream);

}  // namespace fph
