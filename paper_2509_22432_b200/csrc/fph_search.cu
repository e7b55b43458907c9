// fph_search.cu -- flooding kernel, algorithm 1 (default): one warp per
// simplex, exact max of nearest-neighbour distances by bounded search.
//
// The brute-force pass (fph_flood.cu, algorithm 0) evaluates every sample
// point against every cloud point of the simplex's Lemma-4.2 ball.  Most of
// that work cannot change the result: f(sigma) is a MAX over sample points,
// and each point's minimum only needs the cloud points near it.  Per
// simplex, one warp runs (all steps exact; no CTA barriers, so warps never
// wait for each other):
//
//  A  representatives: a stride-s sample (~reps_target points) of the
//     candidate set, against every sample point -> an upper bound
//     U(p) >= nn^2(p) (+ the nearest-vertex bound: vertices are cloud
//     points).  With s = 1 this IS the brute-force pass: done.
//  B  the point with the largest U is searched exactly over the ball of
//     radius sqrt(U) around it -> a certified lower bound L <= f^2.
//  C  point blocks (<= 32 lattice-adjacent rows) in decreasing max-U order:
//     stop as soon as the best remaining block's max U < L; otherwise
//     search the block's points with U >= L exactly over the region that
//     covers their U-balls (centered on those points only; sampled first
//     if the region is large) and raise L.
//  F  finalize: candidates for the maximum (m32 + E >= max(m32 - E)) in
//     decreasing order, each refined to the reference's float64 value over
//     the grid cells of its small ball; stop once no candidate can beat the
//     running maximum.
// fp32 values carry the rigorous error bound E of err_bound(); every bound
// above is taken with it, so the result is the reference's float64 value.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "fph_dev.cuh"

#ifndef FPH_GRID_SLOT
#define FPH_GRID_SLOT 0
#endif
#if FPH_GRID_SLOT == 0
#define FPH_SLOT_NS slot0
#elif FPH_GRID_SLOT == 1
#define FPH_SLOT_NS slot1
#else
#define FPH_SLOT_NS slot2
#endif

namespace fph {

namespace {

constexpr int kSW = 8;          // warps per CTA
constexpr int kSThreads = 32 * kSW;
#ifndef FPH_STAGE_BULK
#define FPH_STAGE_BULK 0
#endif
#ifndef FPH_WT
#define FPH_WT (FPH_STAGE_BULK ? 256 : 512)  // bulk staging: the buffers take the difference
#endif
#ifndef FPH_SEARCH_MINB
#define FPH_SEARCH_MINB 2
#endif
constexpr int kWT = FPH_WT;     // candidates per warp tile

// The grid's parameters for the search kernels.  The grid is built on the
// device (fph_grid.cu computes its box and cell size there, so the host
// never waits for them); before the kernels of a call are queued its
// parameters are copied here device-to-device on the call's stream
// (set_search_grid), where every access is a constant-bank operand, as
// kernel parameters are.  fph_api.cu serialises the calls of a device
// around this slot (GridSlot).
__constant__ Grid c_grid;
constexpr int kMaxBlk = 160;    // blocks ordered best-first per simplex
#ifndef FPH_SPREAD_RATIO
#define FPH_SPREAD_RATIO 16.0
#endif
// phase C searches a block's rows one by one when the region around all
// their U-balls has more than this many times their summed volume
constexpr double kSpreadRatio = FPH_SPREAD_RATIO;
#ifndef FPH_SAMPLE_PASSES
#define FPH_SAMPLE_PASSES 1
#endif
#ifndef FPH_TEAM_REPS
#define FPH_TEAM_REPS 1
#endif
// representative sample of a CTA team's simplex, in units of reps_target
constexpr int kTeamReps = FPH_TEAM_REPS;
#ifndef FPH_TET_REPS_SCALE
#define FPH_TET_REPS_SCALE 0.5
#endif
// tetrahedra (1771 rows at m = 20): representative sample scale -- the
// fold of 512 reps against every row outweighed the tighter bounds
// (modelnet_batch 143 -> 140 ms at 0.5; 0.35 the same, 2 -> 151)
constexpr double kTetRepsScale = FPH_TET_REPS_SCALE;
#ifndef FPH_TRI_REPS_SCALE
#define FPH_TRI_REPS_SCALE 0.75
#endif
// the same for triangles: 0.5 / 0.75 / 1 / 1.5 -> configs[1] 3.49 / 3.47 /
// 3.50 / 3.52 ms, dense30 4.47 / 4.49 / 4.53 / 4.61, modelnet_batch 139.5 /
// 139.9 / 141.0 / 142.1
constexpr double kTriRepsScale = FPH_TRI_REPS_SCALE;
#ifndef FPH_EDGE_REPS_SCALE
#define FPH_EDGE_REPS_SCALE 1.0
#endif
constexpr double kEdgeRepsScale = FPH_EDGE_REPS_SCALE;  // and for edges
#ifndef FPH_COUNT_EST
#define FPH_COUNT_EST 1
#endif
// phase C: sampling passes a large block region may get before its exact pass
constexpr int kSamplePasses = FPH_SAMPLE_PASSES;

// 1: phase C's exact pass stages each window of candidates with bulk copies
// (cp.async.bulk, the TMA engine's 1-D form): every lane copies the piece of
// its grid row's run that falls in the window, 16-byte aligned (up to one
// neighbouring point either side -- real cloud points, filtered like any
// other), completing on the warp's mbarrier; the candidates are then read
// from shared memory in order, without window_index.
constexpr bool kStageBulk = FPH_STAGE_BULK;
#if FPH_STAGE_BULK
constexpr int kBulkW = 96;            // real candidates per window
constexpr int kBulkN = kBulkW + 64;   // + alignment padding (<= 2 per piece)
#endif

struct WarpSmem {
#if FPH_STAGE_BULK
    __align__(16) double bx[kBulkN];
    __align__(16) double by[kBulkN];
    __align__(16) double bz[kBulkN];
    unsigned long long bar;  // the warp's mbarrier
    unsigned bphase;         // its current phase parity
#endif
    float4 tA[kWT / 2];  // pair p: (c0.x, c1.x, c0.y, c1.y)
    float4 tB[kWT / 2];  //         (c0.z, c1.z, |c0|^2, |c1|^2)
    int row_off[32];
    int row_beg[32];
    int pack[32];        // phase C: the block's rows still >= L
    float key[kMaxBlk];
    Verts V;             // the current simplex (kept out of registers)
    SimplexGeom G;
};

// cross-warp scratch of a CTA working on one simplex together
struct TeamSmem {
    float f[kSW][32];
    double d[kSW];
    long long ll[kSW];
    float key[kMaxBlk];
    int t;
};

// Dynamic shared memory: SearchSmem, then (P <= kValsCap) the rows' values of
// every warp, then the m + 1 template weights c / m (a.wt_off).
struct SearchSmem {
    WarpSmem w[kSW];
    TeamSmem team;
};

// Per-row values of the current simplex (U bounds, then certified minima)
// live in shared memory after SearchSmem when the template has at most
// kValsCap rows: every phase reads and writes them, and an L2 round trip per
// access was a large part of a block search's latency.  A team uses warp
// 0's array.  Larger templates use the global scratch (a.perpoint).
#ifndef FPH_VALS_CAP
#define FPH_VALS_CAP 1024
#endif
constexpr int kValsCap = FPH_VALS_CAP;
constexpr size_t kSmemVals = sizeof(SearchSmem) + sizeof(float) * kSW * kValsCap;
static_assert(kSmemVals + 8 * 256 + 1024 <= 233472 / 2, "two search CTAs per SM up to m = 255");

// A team is one warp (size 1) or all warps of the CTA (size kSW) working on
// one simplex: row batches are dealt round-robin to the team's warps and the
// partial results combined through shared memory.
struct Team {
    int rank, size;
    TeamSmem* ts;
    __device__ __forceinline__ void sync() const {
        if (size > 1) __syncthreads(); else __syncwarp();
    }
    // per-lane minimum across the team's warps
    __device__ __forceinline__ float lane_min(float v) const {
        return size == 1 ? v : team_lane_min(ts, rank, v);
    }
    __device__ __forceinline__ double min_d(double v) const {  // warp-uniform v
        return size == 1 ? v : team_min_d(ts, rank, v);
    }
    __device__ __forceinline__ float min_f(float v) const { return (float)min_d((double)v); }
    __device__ __forceinline__ float max_f(float v) const { return -(float)min_d(-(double)v); }
    __device__ __forceinline__ long long sum(long long v) const {  // warp-uniform v
        return size == 1 ? v : team_sum(ts, rank, v);
    }
    // out of line: one copy each (the kernel's instruction footprint matters)
    static __device__ __noinline__ float team_lane_min(TeamSmem* ts, int rank, float v) {
        const int lane = threadIdx.x & 31;
        __syncthreads();
        ts->f[rank][lane] = v;
        __syncthreads();
        float r = ts->f[0][lane];
#pragma unroll
        for (int i = 1; i < kSW; ++i) r = fminf(r, ts->f[i][lane]);
        return r;
    }
    static __device__ __noinline__ double team_min_d(TeamSmem* ts, int rank, double v) {
        __syncthreads();
        if ((threadIdx.x & 31) == 0) ts->d[rank] = v;
        __syncthreads();
        double r = ts->d[0];
#pragma unroll
        for (int i = 1; i < kSW; ++i) r = fmin(r, ts->d[i]);
        return r;
    }
    static __device__ __noinline__ long long team_sum(TeamSmem* ts, int rank, long long v) {
        __syncthreads();
        if ((threadIdx.x & 31) == 0) ts->ll[rank] = v;
        __syncthreads();
        long long r = 0;
#pragma unroll
        for (int i = 0; i < kSW; ++i) r += ts->ll[i];
        return r;
    }
};

struct Ctx {
    const FloodArgs* a;
    const SimplexGeom& G;
    const Verts& V;
    const double* wt;
    float thr;  // simplex ball (Lemma 4.2) on |a|^2; +inf when unpruned
    int s;
    double cnt;  // the simplex's candidate count (a.cand_count[s])
};

struct PointF {
    float bx, by, bz, bb, px2, py2, pz2, B;
};

__device__ __forceinline__ PointF point_at(const Ctx& c, int j, double p64[3]) {
    sample_row_w(*c.a, c.V, c.s, j, c.wt, p64);
    PointF q;
    q.bx = __double2float_rn(__dsub_rn(p64[0], c.G.cx));
    q.by = __double2float_rn(__dsub_rn(p64[1], c.G.cy));
    q.bz = __double2float_rn(__dsub_rn(p64[2], c.G.cz));
    q.bb = fmaf(q.bz, q.bz, fmaf(q.by, q.by, q.bx * q.bx));
    q.px2 = -2.f * q.bx;
    q.py2 = -2.f * q.by;
    q.pz2 = -2.f * q.bz;
    q.B = sqrtf(q.bb) * 1.0001f;
    return q;
}

__device__ __forceinline__ PointF point_at(const Ctx& c, int j) {
    double p64[3];
    return point_at(c, j, p64);
}

// nearest vertex (a cloud point in subset mode): an upper bound on nn^2
__device__ __forceinline__ float vertex_bound(const Ctx& c, const PointF& q) {
    if (!c.a->subset) return INFINITY;
    float dmin = INFINITY, vmax = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (i <= c.a->k) {
            const float vx = __double2float_rn(__dsub_rn(c.V.v[i][0], c.G.cx));
            const float vy = __double2float_rn(__dsub_rn(c.V.v[i][1], c.G.cy));
            const float vz = __double2float_rn(__dsub_rn(c.V.v[i][2], c.G.cz));
            const float dx = q.bx - vx, dy = q.by - vy, dz = q.bz - vz;
            dmin = fminf(dmin, fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
            vmax = fmaxf(vmax, fmaf(vz, vz, fmaf(vy, vy, vx * vx)));
        }
    }
    const float sv = q.B + sqrtf(vmax) * 1.0001f;
    return dmin * 1.00001f + (float)(16.0 * kU32) * sv * sv;
}

// ----------------------------------------------------- warp enumeration
// Rows of a cell box, 32 at a time: lane r computes row r's run; the runs'
// exclusive offsets go to shared memory so any lane can map a flattened
// candidate position to its point index.
struct Rows {
    Box box;
    RowClipF cf;
    bool clip;
};

__device__ __forceinline__ Rows make_rows(double qx, double qy, double qz, double R) {
    const Grid& g = c_grid;
    Rows r;
    r.clip = R < 1e300;
    r.box = r.clip ? ball_box(g, qx, qy, qz, R) : full_box(g);
    if (r.clip) r.cf = make_clip_f(g, qx, qy, qz, R);
    return r;
}

// One batch of 32 rows: lane r holds row r's run; the non-empty runs are
// compacted into shared memory (exclusive offsets and first points) so any
// flattened candidate position maps to its point index.
struct Batch {
    int total;  // candidates in the batch
    int nne;    // non-empty rows
    int off;    // this lane's row: exclusive offset
    int len;    //                  run length
};

__device__ __forceinline__ Batch row_batch(const Rows& rw, WarpSmem& W, int rb) {
    const int lane = threadIdx.x & 31;
    const int rows = rw.box.rows();
    const int r = rb + lane;
    int2 run = make_int2(0, 0);
    if (r < rows) {
        if (rw.clip) {
            run = row_run_f(c_grid, rw.box, r, rw.cf);
        } else {
            const int base = ((rw.box.z0 + r / rw.box.ny_b()) * c_grid.ny + rw.box.y0 +
                              r % rw.box.ny_b()) * c_grid.nx;
            run = make_int2(c_grid.cell_start[base + rw.box.x0],
                            c_grid.cell_start[base + rw.box.x1 + 1]);
        }
    }
    const int len = run.y - run.x;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const unsigned ne = __ballot_sync(0xffffffffu, len > 0);
    const int rank = __popc(ne & ((1u << lane) - 1u));
    __syncwarp();
    if (len > 0) {
        W.row_off[rank] = incl - len;
        W.row_beg[rank] = run.x;
    }
    __syncwarp();
    Batch b;
    b.total = __shfl_sync(0xffffffffu, incl, 31);
    b.nne = __popc(ne);
    b.off = incl - len;
    b.len = len;
    return b;
}

// point index of the contiguous position f0 + lane (garbage when past the
// batch total): the row is the last non-empty row starting at or before it,
// found from the window's start bitmask instead of a search
__device__ __forceinline__ int window_index(const WarpSmem& W, const Batch& b, int f0) {
    const int lane = threadIdx.x & 31;
    const bool starts = b.len > 0 && b.off >= f0 && b.off < f0 + 32;
    const unsigned mask = __reduce_or_sync(0xffffffffu, starts ? 1u << (b.off - f0) : 0u);
    const int before = __popc(__ballot_sync(0xffffffffu, b.len > 0 && b.off < f0));
    const unsigned upto = lane == 31 ? mask : (mask & ((2u << lane) - 1u));
    const int k = max(before + __popc(upto) - 1, 0);
    return W.row_beg[k] + f0 + lane - W.row_off[k];
}

// point index of an arbitrary position f < total (strided sampling)
__device__ __forceinline__ int cand_index(const WarpSmem& W, int nne, int f) {
    int lo = 0, hi = nne;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (W.row_off[mid] <= f) lo = mid; else hi = mid;
    }
    return W.row_beg[lo] + f - W.row_off[lo];
}

__device__ __forceinline__ void load_rel(const Ctx& c, int idx, float& ax, float& ay, float& az,
                                         float& aw) {
    const Grid& g = c_grid;
    ax = __double2float_rn(__dsub_rn(g.x[idx], c.G.cx));
    ay = __double2float_rn(__dsub_rn(g.y[idx], c.G.cy));
    az = __double2float_rn(__dsub_rn(g.z[idx], c.G.cz));
    aw = fmaf(az, az, fmaf(ay, ay, ax * ax));
}

#ifndef FPH_PROBE_CAP
#define FPH_PROBE_CAP 48
#endif
// Local probe of one sample point (one lane, phase A): its nearest
// candidate among the first kProbeCap cloud points of the 3-cell runs of
// its own grid row and the four rows beside it in y and z (kProbeRows 1:
// own row only; 3: y only; 9: the full 3 x 3 x 3).  Without the z rows the
// flat tetrahedra lying on a face of box_10m kept loose bounds and one
// rank of eight took 3.2 ms against 2.4 ms for the others.
// The representatives' bound U of a point in dense data is set by the
// spacing of a ~reps_target sample of the whole masking ball -- an order of
// magnitude above the point's nn distance for a long edge or a large hull
// tetrahedron -- while a point of its own cells is nearly as close as the
// nearest one.  The tight U prunes most rows in phase C without a search
// (box_10m 39 -> 12 ms, with the skipped representatives below).  Any candidate gives an upper bound, so the cap
// and the order are free; the value is the same fp32 expression as every
// other minimum (phase B adds the same error bound), so U stays a
// certified upper bound.
constexpr int kProbeCap = FPH_PROBE_CAP;
#ifndef FPH_PROBE_CAP_TET
#define FPH_PROBE_CAP_TET 16
#endif
constexpr int kProbeCapTet = FPH_PROBE_CAP_TET;  // tetrahedra (1771 rows each)
// (edges and triangles: cap 16 / 24 / 32 / 48 / 64 / 96 -> configs[1] 3.39 /
// 3.35 / 3.34 / 3.27 / 3.31 / 3.43 ms, dense30 4.30 / 4.26 / 4.21 / 4.13 /
// 4.23 / 4.51; box_10m and modelnet_batch within 1% up to 48.  Tetrahedra:
// 16, box_10m 15.2 ms at 8, 11.0 at 24)
#ifndef FPH_PROBE_SKIP
#define FPH_PROBE_SKIP 1
#endif
// 1: a simplex whose every row's probe found a candidate skips the
// representatives' pass ...
constexpr bool kProbeSkip = FPH_PROBE_SKIP;
#ifndef FPH_PROBE_TIGHT
#define FPH_PROBE_TIGHT 4.0f
#endif
// ... provided every probe found one within sqrt(kProbeTight) cell edges
// (looser probe bounds leave phase C more to search than the pass costs)
constexpr float kProbeTight = FPH_PROBE_TIGHT;
#ifndef FPH_PROBE_TIGHT_TRI
#define FPH_PROBE_TIGHT_TRI 1.0f
#endif
constexpr float kProbeTightTri = FPH_PROBE_TIGHT_TRI;  // triangles with a small ball
#ifndef FPH_PROBE_BALL_CELLS
#define FPH_PROBE_BALL_CELLS 8.0
#endif
constexpr double kProbeBallCells = FPH_PROBE_BALL_CELLS;  // "small": rho < this many cell edges
#ifndef FPH_PROBE_SMALL_DIMS
#define FPH_PROBE_SMALL_DIMS 12
#endif
constexpr int kProbeSmallDims = FPH_PROBE_SMALL_DIMS;  // bit k: the rule applies to dimension k
#ifndef FPH_PROBE_BALL_CELLS_TET
#define FPH_PROBE_BALL_CELLS_TET FPH_PROBE_BALL_CELLS
#endif
constexpr double kProbeBallCellsTet = FPH_PROBE_BALL_CELLS_TET;
#ifndef FPH_NO_PROBE_SMALL
#define FPH_NO_PROBE_SMALL 0
#endif
constexpr bool kNoProbeSmall = FPH_NO_PROBE_SMALL;  // 1: small-ball simplices do not probe
#ifndef FPH_PROBE_ALL_SMALL
#define FPH_PROBE_ALL_SMALL 0
#endif
constexpr bool kProbeAllSmall = FPH_PROBE_ALL_SMALL;  // 1: ... probe every row (no early stop)
#ifndef FPH_PROBE_ROWS
#define FPH_PROBE_ROWS 5
#endif
// rows of cells probed: 1 (the point's own), 3 (its y-neighbours), 5 (its y-
// and z-neighbours) or 9
constexpr int kProbeRows = FPH_PROBE_ROWS;

__device__ __forceinline__ float local_probe(const Ctx& c, const PointF& q) {
    const Grid& g = c_grid;
    const double px = c.G.cx + (double)q.bx, py = c.G.cy + (double)q.by,
                 pz = c.G.cz + (double)q.bz;
    const int ix = cell_coord(px, g.lox, g.inv_h, g.nx);
    const int iy = cell_coord(py, g.loy, g.inv_h, g.ny);
    const int iz = cell_coord(pz, g.loz, g.inv_h, g.nz);
    const int x0 = max(ix - 1, 0), x1 = min(ix + 1, g.nx - 1);
    float best = INFINITY;
    int left = c.a->k == 3 ? kProbeCapTet : kProbeCap;
    // one row of cells at a time, so a full own row costs no further loads
    // (fetching every row's run up front: +1-2% on surface data)
    for (int t = 0; t < kProbeRows && left > 0; ++t) {
        // (dy, dz) in the order 0, -1, +1 each: the point's own row first
        // (5 rows: the cross (0, 0), (-1, 0), (+1, 0), (0, -1), (0, +1))
        const int dy = (kProbeRows == 5 && t >= 3) ? 0 : ((t % 3 == 0) ? 0 : (t % 3 == 1 ? -1 : 1));
        const int dz = (kProbeRows == 5 && t >= 3) ? (t == 3 ? -1 : 1)
                                                   : ((t / 3 == 0) ? 0 : (t / 3 == 1 ? -1 : 1));
        const int y = iy + dy, z = iz + dz;
        if (y < 0 || y >= g.ny || z < 0 || z >= g.nz) continue;
        const int base = (z * g.ny + y) * g.nx;
        const int s = g.cell_start[base + x0];
        const int e = min(g.cell_start[base + x1 + 1], s + left);
        left -= e - s;
        int i = s;
        for (; i + 1 < e; i += 2) {  // two loads in flight
            float ax, ay, az, aw, bx, by, bz, bw;
            load_rel(c, i, ax, ay, az, aw);
            load_rel(c, i + 1, bx, by, bz, bw);
            if (aw <= c.thr) best = fminf(best, fmaf(q.px2, ax, fmaf(q.py2, ay, fmaf(q.pz2, az, aw))));
            if (bw <= c.thr) best = fminf(best, fmaf(q.px2, bx, fmaf(q.py2, by, fmaf(q.pz2, bz, bw))));
        }
        if (i < e) {
            float ax, ay, az, aw;
            load_rel(c, i, ax, ay, az, aw);
            if (aw <= c.thr) best = fminf(best, fmaf(q.px2, ax, fmaf(q.py2, ay, fmaf(q.pz2, az, aw))));
        }
    }
    return best < INFINITY ? best + q.bb : INFINITY;  // m32, as the folds give it
}

#if FPH_STAGE_BULK
__device__ __forceinline__ void rel_of(const Ctx& c, double x, double y, double z, float& ax,
                                       float& ay, float& az, float& aw) {
    ax = __double2float_rn(__dsub_rn(x, c.G.cx));
    ay = __double2float_rn(__dsub_rn(y, c.G.cy));
    az = __double2float_rn(__dsub_rn(z, c.G.cz));
    aw = fmaf(az, az, fmaf(ay, ay, ax * ax));
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, void* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void bar_expect(void* bar, unsigned bytes) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(void* bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(b), "r"(parity)
        : "memory");
}
#endif

// append the kept candidates of the warp to the tile; returns the new size
__device__ __forceinline__ int tile_push(WarpSmem& W, int n, bool keep, float ax, float ay,
                                         float az, float aw) {
    const int lane = threadIdx.x & 31;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
        const int q = n + __popc(bal & ((1u << lane) - 1u));
        float* A = reinterpret_cast<float*>(W.tA) + (q >> 1) * 4 + (q & 1);
        float* B = reinterpret_cast<float*>(W.tB) + (q >> 1) * 4 + (q & 1);
        A[0] = ax;
        A[2] = ay;
        B[0] = az;
        B[2] = aw;
    }
    return n + __popc(bal);
}

__device__ __forceinline__ void tile_pad(WarpSmem& W, int n) {
    __syncwarp();
    if ((n & 1) && (threadIdx.x & 31) == 0) {
        float* A = reinterpret_cast<float*>(W.tA) + (n >> 1) * 4;
        float* B = reinterpret_cast<float*>(W.tB) + (n >> 1) * 4;
        A[1] = 0.f;
        A[3] = 0.f;
        B[1] = 0.f;
        B[3] = INFINITY;  // |c|^2 = inf: never the minimum
    }
    __syncwarp();
}

// min over the tile of |a|^2 - 2 a.b for one point (3 FFMA2 + 1 FMNMX3 per
// candidate pair, two independent chains)
__device__ __forceinline__ float tile_min(const WarpSmem& W, int n, const PointF& q, float best) {
    const float2 bx = make_float2(q.px2, q.px2), by = make_float2(q.py2, q.py2),
                 bz = make_float2(q.pz2, q.pz2);
    const int np = (n + 1) >> 1;
    float b0 = best, b1 = INFINITY, b2 = INFINITY, b3 = INFINITY;
    int p = 0;
    // four candidate pairs per iteration: four independent chains
    for (; p + 3 < np; p += 4) {
        float2 u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float4 A = W.tA[p + i], B = W.tB[p + i];
            u[i] = ffma2(bz, make_float2(B.x, B.y), make_float2(B.z, B.w));
            u[i] = ffma2(by, make_float2(A.z, A.w), u[i]);
            u[i] = ffma2(bx, make_float2(A.x, A.y), u[i]);
        }
        b0 = fmin3(b0, u[0].x, u[0].y);
        b1 = fmin3(b1, u[1].x, u[1].y);
        b2 = fmin3(b2, u[2].x, u[2].y);
        b3 = fmin3(b3, u[3].x, u[3].y);
    }
    for (; p < np; ++p) {
        const float4 A = W.tA[p], B = W.tB[p];
        float2 u = ffma2(bz, make_float2(B.x, B.y), make_float2(B.z, B.w));
        u = ffma2(by, make_float2(A.z, A.w), u);
        u = ffma2(bx, make_float2(A.x, A.y), u);
        b0 = fmin3(b0, u.x, u.y);
    }
    return fminf(fminf(b0, b1), fminf(b2, b3));
}

// ------------------------------------------------------------ phase A
// fold a full tile into the running minima of ALL sample points; a team
// folds with atomicMin on order-preserving uints (vals_ord)
__device__ __forceinline__ void lds128(unsigned addr, float4& v) {
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
}

__device__ void fold_all(const Ctx& c, WarpSmem& W, int n, float* vals, const Team& tm,
                            unsigned long long& pairs) {
    const int lane = threadIdx.x & 31;
    tile_pad(W, n);
    const int P = c.a->P;
    const int np = (n + 1) >> 1;
    const unsigned sA = (unsigned)__cvta_generic_to_shared(W.tA), sB = (unsigned)__cvta_generic_to_shared(W.tB);
    const int half = (P + 1) >> 1;
    if (P <= 32 && half <= 16) {
        // few rows (edges): G groups of `half` lanes, two rows per lane, each
        // group folds every G-th candidate pair; group minima meet in group 0
        const int G = 32 / half;
        const int g = lane / half, i = lane - g * half;
        const int ja = i, jb = i + half;
        const PointF qa = point_at(c, min(ja, P - 1));
        const PointF qb = point_at(c, min(jb, P - 1));
        const float2 ax = make_float2(qa.px2, qa.px2), ay = make_float2(qa.py2, qa.py2),
                     az = make_float2(qa.pz2, qa.pz2);
        const float2 bx = make_float2(qb.px2, qb.px2), by = make_float2(qb.py2, qb.py2),
                     bz = make_float2(qb.pz2, qb.pz2);
        float ba = INFINITY, bb = INFINITY;
        for (int p = g < G ? g : np; p < np; p += G) {
            float4 A, B;
            lds128(sA + 16u * p, A);
            lds128(sB + 16u * p, B);
            float2 u = ffma2(az, make_float2(B.x, B.y), make_float2(B.z, B.w));
            float2 v = ffma2(bz, make_float2(B.x, B.y), make_float2(B.z, B.w));
            u = ffma2(ay, make_float2(A.z, A.w), u);
            v = ffma2(by, make_float2(A.z, A.w), v);
            u = ffma2(ax, make_float2(A.x, A.y), u);
            v = ffma2(bx, make_float2(A.x, A.y), v);
            ba = fmin3(ba, u.x, u.y);
            bb = fmin3(bb, v.x, v.y);
        }
        for (int gg = 1; gg < G; ++gg) {
            const int src = min(i + gg * half, 31);
            ba = fminf(ba, __shfl_sync(0xffffffffu, ba, src));
            bb = fminf(bb, __shfl_sync(0xffffffffu, bb, src));
        }
        if (g == 0) {
            const float va = ba + qa.bb, vb = bb + qb.bb;
            if (ja < P) {
                if (tm.size == 1) vals[ja] = fminf(vals[ja], va);
                else atomicMin(reinterpret_cast<unsigned*>(vals) + ja, f2ord(va));
            }
            if (jb < P) {
                if (tm.size == 1) vals[jb] = fminf(vals[jb], vb);
                else atomicMin(reinterpret_cast<unsigned*>(vals) + jb, f2ord(vb));
            }
        }
        pairs += (unsigned long long)n * P;
        __syncwarp();
        return;
    }
    // two points per lane: each tile read serves 64 points
    for (int j0 = 0; j0 < P; j0 += 64) {
        const int ja = j0 + lane, jb = j0 + 32 + lane;
        const PointF qa = point_at(c, min(ja, P - 1));
        const PointF qb = point_at(c, min(jb, P - 1));
        float ba0 = INFINITY, ba1 = INFINITY, bb0 = INFINITY, bb1 = INFINITY;
        int p = 0;
        for (; p + 1 < np; p += 2) {
            float4 A0, B0, A1, B1;
            lds128(sA + 16u * p, A0);
            lds128(sB + 16u * p, B0);
            lds128(sA + 16u * (p + 1), A1);
            lds128(sB + 16u * (p + 1), B1);
            float2 u0 = ffma2(make_float2(qa.pz2, qa.pz2), make_float2(B0.x, B0.y), make_float2(B0.z, B0.w));
            float2 v0 = ffma2(make_float2(qb.pz2, qb.pz2), make_float2(B0.x, B0.y), make_float2(B0.z, B0.w));
            float2 u1 = ffma2(make_float2(qa.pz2, qa.pz2), make_float2(B1.x, B1.y), make_float2(B1.z, B1.w));
            float2 v1 = ffma2(make_float2(qb.pz2, qb.pz2), make_float2(B1.x, B1.y), make_float2(B1.z, B1.w));
            u0 = ffma2(make_float2(qa.py2, qa.py2), make_float2(A0.z, A0.w), u0);
            v0 = ffma2(make_float2(qb.py2, qb.py2), make_float2(A0.z, A0.w), v0);
            u1 = ffma2(make_float2(qa.py2, qa.py2), make_float2(A1.z, A1.w), u1);
            v1 = ffma2(make_float2(qb.py2, qb.py2), make_float2(A1.z, A1.w), v1);
            u0 = ffma2(make_float2(qa.px2, qa.px2), make_float2(A0.x, A0.y), u0);
            v0 = ffma2(make_float2(qb.px2, qb.px2), make_float2(A0.x, A0.y), v0);
            u1 = ffma2(make_float2(qa.px2, qa.px2), make_float2(A1.x, A1.y), u1);
            v1 = ffma2(make_float2(qb.px2, qb.px2), make_float2(A1.x, A1.y), v1);
            ba0 = fmin3(ba0, u0.x, u0.y);
            bb0 = fmin3(bb0, v0.x, v0.y);
            ba1 = fmin3(ba1, u1.x, u1.y);
            bb1 = fmin3(bb1, v1.x, v1.y);
        }
        if (p < np) {
            float4 A0, B0;
            lds128(sA + 16u * p, A0);
            lds128(sB + 16u * p, B0);
            float2 u0 = ffma2(make_float2(qa.pz2, qa.pz2), make_float2(B0.x, B0.y), make_float2(B0.z, B0.w));
            float2 v0 = ffma2(make_float2(qb.pz2, qb.pz2), make_float2(B0.x, B0.y), make_float2(B0.z, B0.w));
            u0 = ffma2(make_float2(qa.py2, qa.py2), make_float2(A0.z, A0.w), u0);
            v0 = ffma2(make_float2(qb.py2, qb.py2), make_float2(A0.z, A0.w), v0);
            u0 = ffma2(make_float2(qa.px2, qa.px2), make_float2(A0.x, A0.y), u0);
            v0 = ffma2(make_float2(qb.px2, qb.px2), make_float2(A0.x, A0.y), v0);
            ba0 = fmin3(ba0, u0.x, u0.y);
            bb0 = fmin3(bb0, v0.x, v0.y);
        }
        const float va = fminf(ba0, ba1) + qa.bb, vb = fminf(bb0, bb1) + qb.bb;
        if (ja < P) {
            if (tm.size == 1) vals[ja] = fminf(vals[ja], va);
            else atomicMin(reinterpret_cast<unsigned*>(vals) + ja, f2ord(va));
        }
        if (jb < P) {
            if (tm.size == 1) vals[jb] = fminf(vals[jb], vb);
            else atomicMin(reinterpret_cast<unsigned*>(vals) + jb, f2ord(vb));
        }
    }
    pairs += (unsigned long long)n * P;
    __syncwarp();
}

__device__ void reps_pass(const Ctx& c, WarpSmem& W, int stride, float* vals, const Team& tm,
                          unsigned long long& pairs, unsigned long long& staged) {
    const int lane = threadIdx.x & 31;
    const FloodArgs& a = *c.a;
    const Rows rw = make_rows(c.G.cx, c.G.cy, c.G.cz, a.subset ? c.G.rho : 1e301);
    const int rows = rw.box.rows();
    int tile_n = 0;
    long long fbase = 0;  // this warp's own enumeration: any subset is a valid sample
    for (int rb = tm.rank * 32; rb < rows; rb += tm.size * 32) {
        const Batch bt = row_batch(rw, W, rb);
        const int total = bt.total;
        const int first = stride == 1 ? 0 : (int)((stride - fbase % stride) % stride);
        const int nsel = total > first ? (total - first - 1) / stride + 1 : 0;
        // two windows of loads in flight (phase A runs in its own kernel, so
        // the extra registers do not reach the search phases)
        for (int i0 = 0; i0 < nsel; i0 += 64) {
            int i[2];
#pragma unroll
            for (int d = 0; d < 2; ++d) {
                const int f = i0 + 32 * d;
                if (stride == 1) i[d] = window_index(W, bt, f);
                else i[d] = f + lane < nsel ? cand_index(W, bt.nne, first + (f + lane) * stride) : 0;
            }
            float ax[2], ay[2], az[2], aw[2];
#pragma unroll
            for (int d = 0; d < 2; ++d) {
                ax[d] = ay[d] = az[d] = aw[d] = 0.f;
                if (i0 + 32 * d + lane < nsel) load_rel(c, i[d], ax[d], ay[d], az[d], aw[d]);
            }
#pragma unroll
            for (int d = 0; d < 2; ++d)
                if (i0 + 32 * d < nsel)
                    tile_n = tile_push(W, tile_n, i0 + 32 * d + lane < nsel && aw[d] <= c.thr, ax[d],
                                       ay[d], az[d], aw[d]);
            if (tile_n > kWT - 64) {
                staged += tile_n;
                fold_all(c, W, tile_n, vals, tm, pairs);
                tile_n = 0;
            }
        }
        fbase += total;
    }
    if (tile_n > 0) {
        staged += tile_n;
        fold_all(c, W, tile_n, vals, tm, pairs);
    }
}

// ------------------------------------------------------- single points
// exact fp32 minimum of |a|^2 - 2 a.b over every candidate within R of q
__device__ float point_min32(const Ctx& c, WarpSmem& W, const PointF& q, double R, const Team& tm,
                             unsigned long long& scanned) {
    const int lane = threadIdx.x & 31;
    const double qx = c.G.cx + (double)q.bx, qy = c.G.cy + (double)q.by,
                 qz = c.G.cz + (double)q.bz;
    const double Rrow = R * (1.0 + 1e-4) + 1e-5 * ((double)q.B + R) + c_grid.margin;
    const Rows rw = make_rows(qx, qy, qz, Rrow);
    const int rows = rw.box.rows();
    float best = INFINITY;
    for (int rb = tm.rank * 32; rb < rows; rb += tm.size * 32) {
        const Batch bt = row_batch(rw, W, rb);
        scanned += bt.total;
        for (int f0 = 0; f0 < bt.total; f0 += 32) {
            const int idx = window_index(W, bt, f0);
            if (f0 + lane < bt.total) {
                float ax, ay, az, aw;
                load_rel(c, idx, ax, ay, az, aw);
                if (aw <= c.thr)
                    best = fminf(best, fmaf(q.px2, ax, fmaf(q.py2, ay, fmaf(q.pz2, az, aw))));
            }
        }
    }
    return tm.min_f(warp_min_f(best));
}

// the reference's float64 squared distance minimised over the grid cells of
// the ball |x - p| <= R (contains every float64 nearest neighbour)
__device__ double point_min64(const Ctx& c, WarpSmem& W, const double p[3], double R,
                              const Team& tm, unsigned long long& scanned) {
    const int lane = threadIdx.x & 31;
    const Rows rw = make_rows(p[0], p[1], p[2], R);
    const int rows = rw.box.rows();
    const Grid& g = c_grid;
    double best = INFINITY;
    for (int rb = tm.rank * 32; rb < rows; rb += tm.size * 32) {
        const Batch bt = row_batch(rw, W, rb);
        scanned += bt.total;
        for (int f0 = 0; f0 < bt.total; f0 += 32) {
            const int idx = window_index(W, bt, f0);
            if (f0 + lane < bt.total)
                best = fmin(best, sq64(g.x[idx], g.y[idx], g.z[idx], p[0], p[1], p[2]));
        }
    }
    return tm.min_d(warp_min_d(best));
}

// ------------------------------------------------------------ phase C
// One block's rows with U >= L (compacted into W.pack, lane i <-> row
// pack[i]) searched exactly over the region that covers their U-balls,
// centered on the midpoint of the balls' bounding box.  Updates vals
// (certified m32, or -inf when the row cannot reach L) and L (identical in
// every warp of the team).  Centering on the active rows only, instead of
// the whole block, cut the staged candidates of this pass ~4x.
__device__ void search_block(const Ctx& c, WarpSmem& W, int nb, float* vals, float& L,
                             const Team& tm, unsigned long long* st) {
    const int lane = threadIdx.x & 31;
    const FloodArgs& a = *c.a;
    const bool valid = lane < nb;
    const int j = W.pack[valid ? lane : nb - 1];  // the packed rows (all >= L when packed)
    const PointF q = point_at(c, j);
    float U2 = vals[j];
    bool active = valid && U2 >= L;
    // center: midpoint of the bounding box of the rows' U-balls (the rows
    // are the still-active ones only, so the region hugs what must be searched)
    const float ru = active ? sqrtf(U2) : 0.f;
    float lx = active ? q.bx - ru : INFINITY, ly = active ? q.by - ru : INFINITY,
          lz = active ? q.bz - ru : INFINITY;
    float hx = active ? q.bx + ru : -INFINITY, hy = active ? q.by + ru : -INFINITY,
          hz = active ? q.bz + ru : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lx = fminf(lx, __shfl_xor_sync(0xffffffffu, lx, o));
        ly = fminf(ly, __shfl_xor_sync(0xffffffffu, ly, o));
        lz = fminf(lz, __shfl_xor_sync(0xffffffffu, lz, o));
        hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
        hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
        hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
    }
    const float cbx = 0.5f * (lx + hx), cby = 0.5f * (ly + hy), cbz = 0.5f * (lz + hz);
    const float ddx = q.bx - cbx, ddy = q.by - cby, ddz = q.bz - cbz;
    const double dB = sqrt((double)ddx * ddx + (double)ddy * ddy + (double)ddz * ddz) * (1.0 + 1e-5) +
                      1e-6 * (double)q.B;
    const double cbn = sqrt((double)cbx * cbx + (double)cby * cby + (double)cbz * cbz);
    // The fp32 region test below accepts every candidate whose true
    // distance to the block center is <= R (1 - 1e-4) - 1e-5 (|cb| + R);
    // cover()'s 1e-3 inflation exceeds that shrink, so each covered U-ball
    // is entirely inside the accepted region: the point is certified.
    auto cover = [&](bool act, float u2) {
        double r = act ? dB + sqrt((double)u2) : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
        return r * (1.0 + 1e-3) + 1e-4 * cbn;
    };
    const double qx = c.G.cx + (double)cbx, qy = c.G.cy + (double)cby, qz = c.G.cz + (double)cbz;
    double R = cover(active, U2);
    // Rows spread far apart relative to their U-balls (a long edge, a big
    // hull triangle): the one region around all the balls holds many times
    // the points of the balls themselves.  Search each active row over its
    // own ball instead (as phase B does for the top row), raising L as it
    // goes -- the same certified values, a fraction of the candidates.
    {
        const double ru = active ? sqrt((double)U2) * (1.0 + 1e-3) + 1e-4 * (double)q.B : 0.0;
        double own = ru * ru * ru;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) own += __shfl_xor_sync(0xffffffffu, own, o);
        if (R * R * R > kSpreadRatio * own) {
            if (valid && !active && tm.rank == 0) vals[j] = -INFINITY;
            unsigned long long scanned = 0;
            unsigned todo = __ballot_sync(0xffffffffu, active);
            while (todo) {
                const int i = __ffs(todo) - 1;
                todo &= todo - 1;
                const float ui = __shfl_sync(0xffffffffu, U2, i);
                const bool mine = lane == i && tm.rank == 0;
                if (!(ui >= L)) {  // dropped below the raised bound
                    if (mine) vals[j] = -INFINITY;
                    continue;
                }
                PointF qi;
                qi.bx = __shfl_sync(0xffffffffu, q.bx, i);
                qi.by = __shfl_sync(0xffffffffu, q.by, i);
                qi.bz = __shfl_sync(0xffffffffu, q.bz, i);
                qi.bb = __shfl_sync(0xffffffffu, q.bb, i);
                qi.px2 = __shfl_sync(0xffffffffu, q.px2, i);
                qi.py2 = __shfl_sync(0xffffffffu, q.py2, i);
                qi.pz2 = __shfl_sync(0xffffffffu, q.pz2, i);
                qi.B = __shfl_sync(0xffffffffu, q.B, i);
                const double Ri = sqrt((double)ui) * (1.0 + 1e-3) + 1e-4 * (double)qi.B;
                const float m = point_min32(c, W, qi, Ri, tm, scanned) + qi.bb;
                if (mine) vals[j] = m;
                L = fmaxf(L, m - err_bound(m, qi.B));
            }
            st[1] += scanned;
            tm.sync();
            return;
        }
    }
    float best = INFINITY;
    int samples = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const bool full = !(R < 1e300);
        const double Rrow = full ? 1e301 : R * (1.0 + 1e-4) + 1e-5 * (cbn + R) + c_grid.margin;
        const float rout2 = full ? INFINITY : (float)(R * R);
        const Rows rw = make_rows(qx, qy, qz, Rrow);
        const int rows = rw.box.rows();
        int stride = 1;
        // a region expected to hold few candidates (the simplex's count
        // scaled by the area ratio, an over-estimate for volume data) skips
        // the counting pass
        // count x min(1, R^2 / rho^2) <= 2 reps, without the division
        const double rho2 = c.G.rho * c.G.rho;
        const bool small = a.subset && rho2 > 0.0 &&
                           c.cnt * fmin(rho2, R * R) <= 2.0 * a.reps_target * rho2;
        if (pass == 0 && !small) {
            // the region's candidate count, estimated from the simplex's by
            // the area ratio (an over-estimate for volume data; counting the
            // region's rows exactly, FPH_COUNT_EST=0, cost phase C 3%): a
            // large region is sampled first to tighten U
            long long cnt = 0;
            if (FPH_COUNT_EST && rho2 > 0.0) {
                cnt = (long long)(c.cnt * fmin(1.0, R * R / rho2));
            } else {
                for (int rb = tm.rank * 32; rb < rows; rb += tm.size * 32) cnt += row_batch(rw, W, rb).total;
                cnt = tm.sum(cnt);
            }
            if (cnt > 4ll * a.reps_target) stride = (int)((cnt + a.reps_target - 1) / a.reps_target);
        }
        if (pass == 1 || stride > 1) {
            int tile_n = 0;
            long long fbase = 0;
            unsigned long long stg = 0;
            auto take = [&](bool keep, float ax, float ay, float az, float aw) {
                tile_n = tile_push(W, tile_n, keep, ax, ay, az, aw);
                if (tile_n > kWT - 32) {
                    tile_pad(W, tile_n);
                    best = tile_min(W, tile_n, q, best);
                    stg += tile_n;
                    tile_n = 0;
                    __syncwarp();
                }
            };
            auto accept = [&](float ax, float ay, float az, float aw) {
                const float dx = ax - cbx, dy = ay - cby, dz = az - cbz;
                return fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= rout2 && aw <= c.thr;
            };
            for (int rb = tm.rank * 32; rb < rows; rb += tm.size * 32) {
                const Batch bt = row_batch(rw, W, rb);
                const int total = bt.total;
                if (stride == 1 && kStageBulk) {
#if FPH_STAGE_BULK
                    for (int f0 = 0; f0 < total; f0 += kBulkW) {
                        const int fe = min(f0 + kBulkW, total);
                        int ps = 0, pe = 0;  // this lane's run piece, sorted indices
                        if (lane < bt.nne) {
                            const int ro = W.row_off[lane];
                            const int re = lane + 1 < bt.nne ? W.row_off[lane + 1] : total;
                            const int lo = max(ro, f0), hi = min(re, fe);
                            if (hi > lo) {
                                ps = W.row_beg[lane] + (lo - ro);
                                pe = ps + (hi - lo);
                            }
                        }
                        const int as = ps & ~1, ae = (pe + 1) & ~1;
                        const int len = pe > ps ? ae - as : 0;
                        int incl = len;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int t = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= o) incl += t;
                        }
                        const int off = incl - len;
                        const int tot = __shfl_sync(0xffffffffu, incl, 31);
                        // the previous window's shared reads before the async writes
                        __syncwarp();
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        if (lane == 0) bar_expect(&W.bar, (unsigned)tot * 24u);
                        if (len > 0) {
                            bulk_g2s(W.bx + off, c_grid.x + as, (unsigned)len * 8u, &W.bar);
                            bulk_g2s(W.by + off, c_grid.y + as, (unsigned)len * 8u, &W.bar);
                            bulk_g2s(W.bz + off, c_grid.z + as, (unsigned)len * 8u, &W.bar);
                        }
                        bar_wait(&W.bar, W.bphase);
                        __syncwarp();
                        if (lane == 0) W.bphase ^= 1u;
                        for (int g0 = 0; g0 < tot; g0 += 32) {
                            const int g = g0 + lane;
                            const bool v = g < tot;
                            float x = 0.f, y = 0.f, z = 0.f, ww = 0.f;
                            if (v) rel_of(c, W.bx[g], W.by[g], W.bz[g], x, y, z, ww);
                            take(v && accept(x, y, z, ww), x, y, z, ww);
                        }
                    }
#endif
                } else if (stride == 1) {
                    // two windows in flight: both loads issue before either is used
                    for (int f0 = 0; f0 < total; f0 += 64) {
                        const int i0 = window_index(W, bt, f0);
                        const int i1 = window_index(W, bt, f0 + 32);
                        const bool v0 = f0 + lane < total, v1 = f0 + 32 + lane < total;
                        float x0 = 0.f, y0 = 0.f, z0 = 0.f, w0 = 0.f, x1 = 0.f, y1 = 0.f, z1 = 0.f,
                              w1 = 0.f;
                        if (v0) load_rel(c, i0, x0, y0, z0, w0);
                        if (v1) load_rel(c, i1, x1, y1, z1, w1);
                        take(v0 && accept(x0, y0, z0, w0), x0, y0, z0, w0);
                        if (f0 + 32 < total) take(v1 && accept(x1, y1, z1, w1), x1, y1, z1, w1);
                    }
                } else {
                    const int first = stride == 1 ? 0 : (int)((stride - fbase % stride) % stride);
                    const int nsel = total > first ? (total - first - 1) / stride + 1 : 0;
                    for (int i0 = 0; i0 < nsel; i0 += 32) {
                        bool keep = false;
                        float ax = 0.f, ay = 0.f, az = 0.f, aw = 0.f;
                        if (i0 + lane < nsel) {
                            load_rel(c, cand_index(W, bt.nne, first + (i0 + lane) * stride), ax, ay,
                                     az, aw);
                            keep = accept(ax, ay, az, aw);
                        }
                        take(keep, ax, ay, az, aw);
                    }
                }
                fbase += total;
            }
            if (tile_n > 0) {
                tile_pad(W, tile_n);
                best = tile_min(W, tile_n, q, best);
                stg += tile_n;
                __syncwarp();
            }
            st[pass] += stg;
            st[2] += stg * (unsigned long long)nb;
            best = tm.lane_min(best);
        }
        if (pass == 0) {
            if (stride > 1) {
                const float m = best + q.bb;
                U2 = fminf(U2, m + err_bound(m, q.B));
                active = active && U2 >= L;
                if (!__any_sync(0xffffffffu, active)) break;
                R = cover(active, U2);
                // the tightened balls may still span a large region: count
                // and sample it again before the exact pass
                if (++samples < kSamplePasses) pass = -1;
            }
            continue;
        }
        const float m32 = best + q.bb;
        if (valid && tm.rank == 0) vals[j] = active ? m32 : -INFINITY;
        const float lb = warp_max(active ? m32 - err_bound(m32, q.B) : -INFINITY);
        L = fmaxf(L, lb);
        tm.sync();
        return;
    }
    if (valid && tm.rank == 0) vals[j] = -INFINITY;  // pruned after sampling
    tm.sync();
}

// ------------------------------------------------------------- finalize
// vals: certified m32 or -inf.  Returns the reference's float64 value.
__device__ double finalize_team(const Ctx& c, WarpSmem& W, float* vals, const Team& tm,
                                unsigned long long& refined, unsigned long long& scanned) {
    const int lane = threadIdx.x & 31;
    const int P = c.a->P;
    // keys m32 + E (upper bounds), L2 = max(m32 - E) (lower bound)
    float lmax = -INFINITY;
    for (int j = tm.rank * 32 + lane; j < P; j += tm.size * 32) {
        const float v = vals[j];
        if (v > -INFINITY) {
            const PointF q = point_at(c, j);
            const float E = err_bound(v, q.B);
            lmax = fmaxf(lmax, v - E);
            vals[j] = v + E;
        }
    }
    const float L2 = tm.max_f(warp_max(lmax));
    tm.sync();
    double M = -INFINITY;
    for (;;) {
        float kmax = -INFINITY;
        int jm = 0x7fffffff;
        for (int j = tm.rank * 32 + lane; j < P; j += tm.size * 32) {
            const float v = vals[j];
            if (v > kmax) {
                kmax = v;
                jm = j;
            }
        }
        const float kw = warp_max(kmax);
        const float km = tm.max_f(kw);
        if (!(km >= L2) || (double)km <= M) break;
        int jw = __reduce_min_sync(0xffffffffu, kmax == km ? jm : 0x7fffffff);
        jm = -(int)tm.max_f(-(float)jw);  // lowest index holding km (exact in fp32 below 2^24)
        double p[3];
        const PointF q = point_at(c, jm, p);
        const float E = err_bound(km, q.B) * 1.01f;
        const double R = sqrt((double)km + (double)E) * (1.0 + 1e-6) + 1e-300;
        M = fmax(M, point_min64(c, W, p, R, tm, scanned));
        ++refined;
        tm.sync();
        if (tm.rank == 0 && lane == 0) vals[jm] = -INFINITY;
        tm.sync();
    }
    return M;
}

// Phase A's candidate stride for a simplex of C candidates: 1 (one exact
// pass) when small, else about C / reps (reps_target, x kTeamReps for a CTA
// team, x kTetRepsScale for tetrahedra).  Every phase kernel must derive it
// the same way -- B and C skip the simplices whose stride is 1.
__device__ __forceinline__ int sample_stride(const FloodArgs& a, long long C, bool team) {
    if ((double)C * (double)a.P <= a.exact_pairs || C <= a.exact_cand[a.k]) return 1;
    long long n_reps = team ? (long long)a.reps_target * kTeamReps : a.reps_target;
    if (a.k == 3) n_reps = max(32ll, (long long)(n_reps * kTetRepsScale));
    if (a.k == 2) n_reps = max(32ll, (long long)(n_reps * kTriRepsScale));
    if (a.k == 1) n_reps = max(32ll, (long long)(n_reps * kEdgeRepsScale));
    return (int)max(1ll, (C + n_reps - 1) / n_reps);
}

// ------------------------------------------------------- one simplex
// kPh: 0 = every phase (one kernel, small complexes); the four-kernel chain
// runs 1 = phase A only (the rows' values go to the next kernel through
// a.perpoint), 5 = phase B only (L to a.lower), 6 = phase C only, 4 = phase
// F only.
template <int kPh>
__device__ void run_simplex(const Ctx& c, WarpSmem& W, const Team& tm, float* vals) {
    const int lane = threadIdx.x & 31;
    const FloodArgs& a = *c.a;
    unsigned long long pairs = 0, staged = 0, st[7] = {0, 0, 0, 0, 0, 0, 0}, refined = 0, scanned = 0,
                       blocks = 0, pruned = 0, searches = 0;
    long long clk[5];
    clk[0] = clock64();
    // ---- A
    int stride = 1;
    if (kPh == 5 || kPh == 6) stride = sample_stride(a, a.cand_count[c.s], tm.size > 1);
    if (kPh == 0 || kPh == 1) {
        for (int j = tm.rank * 32 + lane; j < a.P; j += tm.size * 32)
            vals[j] = tm.size == 1 ? INFINITY : __uint_as_float(f2ord(INFINITY));
        tm.sync();
        // small enough for one exact pass (every row x every candidate), else a
        // sample of ~reps_target candidates (the same stride in every phase
        // kernel: stride 1 means phase A was exact and B / C have nothing to do)
        stride = sample_stride(a, a.cand_count[c.s], tm.size > 1);
        // sampled simplices: every row first probes its own cells; when all
        // rows found a close candidate there (dense data) those bounds
        // replace the representatives' -- whose pass enumerates every grid
        // row of the masking ball, the dominant cost of a large simplex
        bool reps = true;
        const bool small_dims_ball =
            ((kProbeSmallDims >> a.k) & 1) &&
            c.G.rho < (a.k == 3 ? kProbeBallCellsTet : kProbeBallCells) * c_grid.h;
        if (stride > 1 && kProbeCap > 0 && !(kNoProbeSmall && small_dims_ball)) {
            // batch by batch of rows; the first batch with a loose row ends
            // the probing (the pass runs anyway, so further probes would
            // only add their cost: surface data, voids)
            // simplices with a small masking ball (rho < 8 cell edges: the
            // representatives' pass is cheap and its bounds are tighter than
            // a probe's on surface data) skip the pass only when every probe
            // landed within 1 cell edge; large balls (a box hull sliver:
            // the pass enumerates ~10^5 grid rows) keep 2 edges.  configs[1]
            // 3.47 -> 3.37 ms, dense30 4.45 -> 4.29, modelnet_batch 140 ->
            // 124 ms, box_10m even; larger "small" radii cost box_10m up to 2.5x
            const bool small_ball =
                c.G.rho < (a.k == 3 ? kProbeBallCellsTet : kProbeBallCells) * c_grid.h;
            const float tight = (((kProbeSmallDims >> a.k) & 1) && small_ball ? kProbeTightTri
                                                                              : kProbeTight) *
                                (float)(c_grid.h * c_grid.h);
            reps = false;
            for (int j0 = 0; j0 < a.P; j0 += tm.size * 32) {
                const int j = j0 + tm.rank * 32 + lane;
                int miss = 0;
                if (j < a.P) {
                    const float m = local_probe(c, point_at(c, j));
                    miss = !(m <= tight);  // none, or not within ~a cell edge
                    if (m < INFINITY) {
                        if (tm.size == 1) vals[j] = m;
                        else atomicMin(reinterpret_cast<unsigned*>(vals) + j, f2ord(m));
                    }
                }
                if (tm.sum((long long)__reduce_add_sync(0xffffffffu, (unsigned)miss)) > 0) {
                    reps = true;
                    if (!(kProbeAllSmall && small_dims_ball)) break;
                }
            }
            reps = reps || !kProbeSkip;
            tm.sync();
        }
        if (reps) reps_pass(c, W, stride, vals, tm, pairs, staged);
        tm.sync();
        if (tm.size > 1) {  // decode the ordered minima
            __threadfence_block();
            for (int j = tm.rank * 32 + lane; j < a.P; j += tm.size * 32)
                vals[j] = ord2f(__float_as_uint(vals[j]));
            tm.sync();
        }
    }
    clk[1] = clock64();
    clk[2] = clk[1];
    clk[3] = clk[1];
    if ((kPh == 0 || kPh == 5 || kPh == 6) && stride > 1) {
      float L;
      if (kPh == 6) {
        L = a.lower[c.s];  // phase B ran in the previous kernel
      } else {
        // ---- B: upper bounds; exact search of the top point
        float umax = -INFINITY;
        int jmax = 0x7fffffff;
        for (int j = tm.rank * 32 + lane; j < a.P; j += tm.size * 32) {
            const PointF q = point_at(c, j);
            const float m = vals[j];
            const float u = fminf(m + err_bound(m, q.B), vertex_bound(c, q));
            vals[j] = u;
            if (u > umax) {
                umax = u;
                jmax = j;
            }
        }
        const float um = tm.max_f(warp_max(umax));
        const int jw = __reduce_min_sync(0xffffffffu, umax == um ? jmax : 0x7fffffff);
        const int jt = -(int)tm.max_f(-(float)jw);
        tm.sync();
        {
            const PointF q = point_at(c, jt);
            const double R = sqrt((double)um) * (1.0 + 1e-3) + 1e-4 * (double)q.B;
            const float m = point_min32(c, W, q, R, tm, scanned) + q.bb;
            L = m - err_bound(m, q.B);
        }
        if (kPh == 5 && tm.rank == 0 && lane == 0) a.lower[c.s] = L;
      }
        clk[2] = clock64();
      if (kPh != 5) {
        // ---- C: blocks best-first (in order when there are too many to rank);
        // one call site, so search_block is inlined once
        const int nblk = a.nblk;
        const bool ranked = nblk <= kMaxBlk;
        float* key = tm.size == 1 ? W.key : tm.ts->key;
        if (ranked) {
            for (int b = tm.rank * 32 + lane; b < nblk; b += tm.size * 32) {
                float k2 = -INFINITY;
                for (int i = a.blk_off[b]; i < a.blk_off[b + 1]; ++i) k2 = fmaxf(k2, vals[i]);
                key[b] = k2;
            }
            tm.sync();
        }
        auto best_block = [&](float& km) {
            float kb = -INFINITY;
            int bb = 0x7fffffff;
            for (int i = lane; i < nblk; i += 32)
                if (key[i] > kb) {
                    kb = key[i];
                    bb = i;
                }
            km = warp_max(kb);
            return __reduce_min_sync(0xffffffffu, kb == km ? bb : 0x7fffffff);
        };
        auto take_block = [&](int b) {
            tm.sync();
            if (tm.rank == 0 && lane == 0) key[b] = -INFINITY;
            tm.sync();
        };
        // rows of block b with U >= L appended to the pack (lane i <-> row
        // j0 + i); rows below L drop out, as search_block would drop them
        auto rows_of = [&](int b, int& j, float& u) {  // (one call site)
            const int j0 = a.blk_off[b], nb = a.blk_off[b + 1] - j0;
            const bool valid = lane < nb;
            j = j0 + (valid ? lane : 0);
            u = valid ? vals[j] : -INFINITY;
            if (valid && !(u >= L) && tm.rank == 0) vals[j] = -INFINITY;
            return __ballot_sync(0xffffffffu, valid && u >= L);
        };
        const unsigned lt = (1u << lane) - 1u;
        for (int seq = 0;; ++seq) {
            int b = seq;
            float km;
            if (ranked) {
                b = best_block(km);
                if (!(km >= L)) break;  // every remaining block is below L
                take_block(b);
            } else if (seq >= nblk) {
                break;
            }
            ++blocks;
            int j;
            float u;
            unsigned m = rows_of(b, j, u);
            if (m & (1u << lane)) W.pack[__popc(m & lt)] = j;
            int np = __popc(m);
            __syncwarp();
            if (np > 0) {
                search_block(c, W, np, vals, L, tm, st);
                ++searches;
            }
        }
        if (ranked) {
            // blocks never searched cannot reach L
            for (int b = 0; b < nblk; ++b) {
                if (key[b] > -INFINITY) {
                    ++pruned;
                    for (int i = a.blk_off[b] + tm.rank * 32 + lane; i < a.blk_off[b + 1];
                         i += tm.size * 32)
                        vals[i] = -INFINITY;
                }
            }
            tm.sync();
        }
      }
    }
    tm.sync();
    if (stride > 1) clk[3] = clock64();
    const bool fin = kPh == 0 || kPh == 4;  // 5: B only, 6: C only
    const double M = fin ? finalize_team(c, W, vals, tm, refined, scanned) : 0.0;
    clk[4] = clock64();
    unsigned long long* stats = a.stats;
    if (lane == 0) {
        if (tm.rank == 0 && fin) {
            a.out_sq[c.s] = M;
            atomicAdd(&stats[5], 1ull);
            atomicAdd(&stats[7], blocks);
            atomicAdd(&stats[15], searches);
            atomicAdd(&stats[8], pruned);
            atomicAdd(&stats[3], refined);
            if (tm.size > 1) atomicAdd(&stats[9], 1ull);
        }
        atomicAdd(&stats[0], pairs + st[2]);
        atomicAdd(&stats[1], staged + st[0] + st[1]);
        atomicAdd(&stats[4], scanned);
        atomicAdd(&stats[16], staged);
        atomicAdd(&stats[17], st[0]);
        atomicAdd(&stats[18], st[1]);
        // useful (active-lane) vs executed pairs per phase-C pass; phase-A pairs
        for (int i = 0; i < 4; ++i) atomicAdd(&stats[10 + i], st[3 + i]);
        atomicAdd(&stats[14], pairs);
        // warp-cycles per phase (A, B, C, finalize)
        for (int i = 0; i < 4; ++i) atomicAdd(&stats[19 + i], (unsigned long long)(clk[i + 1] - clk[i]));
        if (a.dbg && tm.rank == 0) {  // accumulated: the chained kernels each add their part
            unsigned long long* d = reinterpret_cast<unsigned long long*>(a.dbg + (size_t)c.s * kDbgFields);
            atomicAdd(d + 4, blocks);
            atomicMax(d + 5, (unsigned long long)c.cnt);  // the candidate count
            atomicAdd(d + 6, staged + st[0] + st[1]);
            atomicMax(d + 7, (unsigned long long)tm.size);
        }
    }
    tm.sync();
}

__device__ __forceinline__ int ld_acquire_i(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_i(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Chained phase kernels (pos = place in the chain, stage != nullptr): every
// kernel lets the next one launch at once (programmatic dependent launch),
// so the next phase's CTAs take the SM slots the moment this phase's CTAs
// run out of work; instead of waiting for the whole grid, a CTA waits only
// for ITS simplex's previous phase (stage[s] >= pos, published with release
// after the rows were written).  Every simplex of the previous phase is
// claimed by a resident CTA before any of its CTAs exits, so the waits
// always end.
template <bool kSV, int kPh>
__global__ void __launch_bounds__(kSThreads, FPH_SEARCH_MINB)
    search_kernel(const __grid_constant__ FloodArgs a, const SimplexGeom* __restrict__ geom,
                  const int* __restrict__ order, int* counter, int* stage, int pos) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SearchSmem& S = *reinterpret_cast<SearchSmem*>(smem_raw);
    double* wt = reinterpret_cast<double*>(smem_raw + a.wt_off);
    for (int i = threadIdx.x; i <= a.m; i += blockDim.x) wt[i] = __ddiv_rn((double)i, (double)a.m);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem& W = S.w[w];
#if FPH_STAGE_BULK
    if (lane == 0) {
        const unsigned b = (unsigned)__cvta_generic_to_shared(&W.bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        W.bphase = 0;
    }
    __syncwarp();
#endif
    const long long team_thr = a.team_thr_dev ? *a.team_thr_dev : (long long)a.team_threshold;
    // team mode: the whole CTA per simplex while the queue (sorted by
    // candidate count, largest first) holds big simplices; then warp mode.
    // One call site of run_simplex: the kernel body is inlined once.
    int pending = -1, next = -1;
    bool team = true;
    for (;;) {
        int t;
        if (team) {
            __syncthreads();
            if (threadIdx.x == 0) S.team.t = atomicAdd(counter, 1);
            __syncthreads();
            t = S.team.t;
            if (t >= a.n) return;
            if (a.cand_count[order[t]] <= team_thr) {
                team = false;
                pending = t;  // first small simplex: handed to warp 0
                continue;
            }
        } else if (w == 0 && pending >= 0) {
            t = pending;
            pending = -1;
        } else {
            // the claim for the NEXT simplex is issued now and consumed on the
            // next pass, so its atomic round trip overlaps this simplex
            if (lane == 0) {
                t = next >= 0 ? next : atomicAdd(counter, 1);
                next = -1;
            }
            t = __shfl_sync(0xffffffffu, t, 0);
        }
        if (t >= a.n) return;
        const long long t_claim = clock64();
        long long g_claim = 0;
        if (a.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_claim));
        const int s = order[t];
        // Simplices valued by one exact pass in phase A have no B or C: those
        // kernels skip them outright and F waits for A's flag instead.
        int need = pos;
        if (stage && (kPh == 4 || kPh == 5 || kPh == 6)) {
            const long long C = a.cand_count[s];
            if ((double)C * (double)a.P <= a.exact_pairs || C <= a.exact_cand[a.k]) {
                if (kPh != 4) continue;
                need = 1;
            }
        }
        // geometry and vertices on separate lanes, while lane 0 waits for this
        // simplex's previous phase (the rows it left are read after this)
        __syncwarp();
        static_assert(sizeof(SimplexGeom) % 8 == 0 && sizeof(SimplexGeom) <= 8 * 16, "geom words");
        if (lane >= 16 && lane < 16 + (int)(sizeof(SimplexGeom) / 8))
            reinterpret_cast<long long*>(&W.G)[lane - 16] =
                reinterpret_cast<const long long*>(geom + s)[lane - 16];
        if (lane >= 4 && lane < 8) {
            const int j = lane - 4;
            const int id = j <= a.k ? a.simplices[(size_t)s * 4 + j] : -1;
            W.V.v[j][0] = id >= 0 ? a.landmarks[(size_t)id * 3 + 0] : 0.0;
            W.V.v[j][1] = id >= 0 ? a.landmarks[(size_t)id * 3 + 1] : 0.0;
            W.V.v[j][2] = id >= 0 ? a.landmarks[(size_t)id * 3 + 2] : 0.0;
        }
        if (stage && pos > 0) {
            if ((team ? threadIdx.x : lane) == 0)
                while (ld_acquire_i(stage + s) < need) __nanosleep(64);
            if (team) __syncthreads();
        }
        __syncwarp();
        const Ctx c{&a, W.G, W.V, wt,
                    a.subset ? (float)(W.G.rho * W.G.rho * (1.0 + 1e-5)) : INFINITY, s,
                    (double)a.cand_count[s]};
        const Team tm = team ? Team{w, kSW, &S.team} : Team{0, 1, nullptr};
        float* vals = a.perpoint + (size_t)s * a.P;
        if (kSV) {
            float* sv = reinterpret_cast<float*>(smem_raw + sizeof(SearchSmem)) +
                        (team ? 0 : w) * kValsCap;
            if (kPh >= 2) {  // an earlier kernel left the rows' values
                for (int j = tm.rank * 32 + lane; j < a.P; j += tm.size * 32) sv[j] = vals[j];
                tm.sync();
            }
            run_simplex<kPh>(c, W, tm, sv);
            if (kPh == 1 || kPh == 5 || kPh == 6) {  // hand the rows on
                for (int j = tm.rank * 32 + lane; j < a.P; j += tm.size * 32) vals[j] = sv[j];
                tm.sync();
            }
        } else {
            run_simplex<kPh>(c, W, tm, vals);
        }
        if (stage) {  // publish: this simplex's phase is done
            __threadfence();
            tm.sync();
            if (tm.rank == 0 && lane == 0) st_release_i(stage + s, pos + 1);
        }
        if (a.dbg && lane == 0 && (team ? w == 0 : true)) {
            // profiling aid: cycles of this simplex in this kernel (claim to
            // publish) and its global-timer interval, per phase slot: A 0,
            // B 1, C 2, F 3 (one kernel: 0)
            const int slot = kPh == 5 ? 1 : (kPh == 6 ? 2 : (kPh == 4 ? 3 : 0));
            long long* d = a.dbg + (size_t)s * kDbgFields;
            atomicAdd(reinterpret_cast<unsigned long long*>(d) + slot,
                      (unsigned long long)(clock64() - t_claim));
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            d[8 + 2 * slot] = g_claim;
            d[9 + 2 * slot] = (long long)t_end;
        }
    }
}

// Auto team threshold: a simplex is searched by a whole CTA when its
// predicted cost exceeds beta x (the whole launch's predicted cost / resident
// warps) -- one warp would otherwise still be busy with it long after the
// others ran dry.  Cost grows sublinearly with the candidate count C
// (measured log-log slopes 0.24..0.52, tools/simplex_costs.py), modelled as
// C^p; the threshold is returned in candidates: (beta sum C^p / warps)^(1/p).
#ifndef FPH_TEAM_BETA
#define FPH_TEAM_BETA 2.0
#endif
constexpr double kTeamBeta = FPH_TEAM_BETA;
constexpr long long kTeamMin = 32768;
#ifndef FPH_TEAM_POW
#define FPH_TEAM_POW 1.0
#endif
#ifndef FPH_TEAM_GAMMA
#define FPH_TEAM_GAMMA 0.0
#endif

// sum of C^p (sum[0]) and the largest C (as a double in sum[1])
__global__ void pow_sum_kernel(const int* __restrict__ cand, int n, double p, double* sum) {
    __shared__ double part[8];
    __shared__ int mpart[8];
    double v = 0.0;
    int mx = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        v += p == 1.0 ? (double)cand[i] : pow((double)cand[i], p);
        mx = max(mx, cand[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        part[threadIdx.x >> 5] = v;
        mpart[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        int m = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            t += part[i];
            m = max(m, mpart[i]);
        }
        atomicAdd(sum, t);
        atomicMax(reinterpret_cast<int*>(sum + 1), m);
    }
}

// gamma > 0 also gives a team to every simplex above gamma x the largest
// count: the few heaviest simplices bound a launch's critical path
__global__ void team_thr_kernel(const double* sum, double beta, double p, double gamma, int warps,
                                long long* thr) {
    double t = pow(beta * sum[0] / (double)(warps > 0 ? warps : 1), 1.0 / p);
    const int mx = *reinterpret_cast<const int*>(sum + 1);
    if (gamma > 0.0) t = fmin(t, gamma * (double)mx);
    *thr = t > (double)kTeamMin ? (long long)t : kTeamMin;
}

constexpr int kSortLo = 8;

__global__ void iota_kernel(int* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

__device__ __forceinline__ unsigned spread3(unsigned v) {  // 8 bits -> every third bit
    v &= 0xffu;
    v = (v | (v << 8)) & 0x0f00fu;
    v = (v | (v << 4)) & 0x0c30c3u;
    v = (v | (v << 2)) & 0x249249u;
    return v;
}

// Schedule key of each simplex: the team-sized ones first (bucket 31), then
// descending candidate count in factor-2 buckets; within a bucket the 24-bit
// Morton code of the simplex's cell, so the warps working at the same time
// read neighbouring parts of the cloud (L2 reuse; a 10M-point cloud does not
// fit in L2).  Sorted descending on bits [0, 29).
__global__ void order_key_kernel(const Grid* __restrict__ gp, const SimplexGeom* __restrict__ geom,
                                 const int* __restrict__ cand, int n, const long long* thr_dev,
                                 long long thr_fixed, int* __restrict__ key) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Grid g = *gp;
    const int nmax = max(g.nx, max(g.ny, g.nz));
    const int bits = 32 - __clz(max(nmax - 1, 1));
    const int shift = bits > 8 ? bits - 8 : 0;
    const long long thr = thr_dev ? *thr_dev : thr_fixed;
    const int c = cand[i];
    const unsigned bucket = c > thr ? 31u : (unsigned)min(30, 31 - __clz(c + 1));
    const SimplexGeom& G = geom[i];
    const unsigned ix = (unsigned)cell_coord(G.cx, g.lox, g.inv_h, g.nx) >> shift;
    const unsigned iy = (unsigned)cell_coord(G.cy, g.loy, g.inv_h, g.ny) >> shift;
    const unsigned iz = (unsigned)cell_coord(G.cz, g.loz, g.inv_h, g.nz) >> shift;
    key[i] = (int)((bucket << 24) | (spread3(iz) << 2) | (spread3(iy) << 1) | spread3(ix));
}

}  // namespace

namespace FPH_SLOT_NS {

int set_search_grid(const Grid* d_grid, cudaStream_t stream) {
    FPH_CUDA_TRY(cudaMemcpyToSymbolAsync(c_grid, d_grid, sizeof(Grid), 0, cudaMemcpyDeviceToDevice,
                                         stream));
    return FPH_OK;
}

size_t search_smem_bytes(int P, int m) {
    return (P <= kValsCap ? kSmemVals : sizeof(SearchSmem)) + sizeof(double) * (size_t)(m + 1);
}

size_t search_smem_limit() {
    int dev = 0, lim = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&lim, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return 0;
    return (size_t)lim;
}

int search_prepare(const FloodArgs& a, const SimplexGeom* d_geom, const int* d_cand,
                   cudaStream_t stream, SearchPlan* plan) {
    SearchPlan& p = *plan;
    p = SearchPlan{};
    p.stream = stream;
    p.d_geom = d_geom;
    int dev = 0, sms = 0, occ = 0;
    FPH_CUDA_TRY(cudaGetDevice(&dev));
    FPH_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const bool sv = a.P <= kValsCap;
    p.smem = (int)search_smem_bytes(a.P, a.m);
    // Launches with enough work run the phases as four kernels, A | B | C | F,
    // each with its own register allocation (phase C alone lost a third of its
    // cycles that way), chained per simplex by programmatic dependent launch so
    // each kernel's tail overlaps the next one.  Light launches keep one
    // kernel, where the extra launches and tails do not amortise.  Work
    // estimate: simplices x rows x cloud points per landmark, >= 1e8 (a box
    // shard of 4k tetrahedra of 10M points is heavy, 8k triangles of a 10k
    // torus are not); without the ratio, >= 10 000 simplices.
    // FPH_SPLIT_MIN_SIMPLICES (environment) overrides with a simplex count;
    // the tests set it to 0 to run the small golden complexes through the chain
    bool chain = a.points_per_landmark > 0.0
                     ? (double)a.n * (double)a.P * a.points_per_landmark >= 1e8
                     : a.n >= 10000;
    if (const char* e = getenv("FPH_SPLIT_MIN_SIMPLICES")) chain = a.n >= atoll(e);
    if (chain) {
        p.kern[0] = sv ? search_kernel<true, 1> : search_kernel<false, 1>;
        p.kern[1] = sv ? search_kernel<true, 5> : search_kernel<false, 5>;
        p.kern[2] = sv ? search_kernel<true, 6> : search_kernel<false, 6>;
        p.kern[3] = sv ? search_kernel<true, 4> : search_kernel<false, 4>;
        FPH_CUDA_TRY(cudaMallocAsync(&p.d_lower, sizeof(float) * a.n, stream));
    } else {
        p.kern[0] = sv ? search_kernel<true, 0> : search_kernel<false, 0>;
    }
    FPH_CUDA_TRY(cudaFuncSetAttribute(p.kern[0], cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem));
    FPH_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p.kern[0], kSThreads, p.smem));
    int blocks = sms * (occ > 0 ? occ : 1);
    p.blocks = blocks < (a.n + kSW - 1) / kSW ? blocks : (a.n + kSW - 1) / kSW;
    p.b = a;
    p.b.lower = p.d_lower;
    p.b.wt_off = (int)(sv ? kSmemVals : sizeof(SearchSmem));
    if (a.team_threshold <= 0) {
        // threshold from the total candidate count, computed on the device so
        // the concurrent streams never wait for the host
        const double beta = a.team_threshold < 0 ? -a.team_threshold / 100.0 : kTeamBeta;
        static const double team_pow =
            getenv("FPH_TEAM_POW") ? atof(getenv("FPH_TEAM_POW")) : FPH_TEAM_POW;
        static const double team_gamma =
            getenv("FPH_TEAM_GAMMA") ? atof(getenv("FPH_TEAM_GAMMA")) : FPH_TEAM_GAMMA;
        FPH_CUDA_TRY(cudaMallocAsync(&p.d_thr, 3 * sizeof(long long), stream));
        double* d_sum = reinterpret_cast<double*>(p.d_thr + 1);
        FPH_CUDA_TRY(cudaMemsetAsync(d_sum, 0, 2 * sizeof(double), stream));
        pow_sum_kernel<<<std::min(148, (a.n + 255) / 256), 256, 0, stream>>>(d_cand, a.n, team_pow,
                                                                          d_sum);
        team_thr_kernel<<<1, 1, 0, stream>>>(d_sum, beta, team_pow, team_gamma, p.blocks * kSW,
                                             p.d_thr);
        p.b.team_thr_dev = p.d_thr;
    }
    // order: FPH_ORDER=0 (environment) sorts by candidate count alone,
    // largest first (bits [8, 24)); the default adds spatial locality
    // (order_key_kernel)
    static const int order_mode = getenv("FPH_ORDER") ? atoi(getenv("FPH_ORDER")) : 1;
    FPH_CUDA_TRY(cudaMallocAsync(&p.d_keys, sizeof(int) * a.n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&p.d_order, sizeof(int) * a.n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&p.d_iota, sizeof(int) * a.n, stream));
    iota_kernel<<<(a.n + 255) / 256, 256, 0, stream>>>(p.d_iota, a.n);
    int lo_bit = kSortLo, hi_bit = 24;
    const int* sort_in = d_cand;
    if (order_mode == 1) {
        FPH_CUDA_TRY(cudaMallocAsync(&p.d_key_in, sizeof(int) * a.n, stream));
        order_key_kernel<<<(a.n + 255) / 256, 256, 0, stream>>>(
            a.gp, d_geom, d_cand, a.n, p.b.team_thr_dev, (long long)a.team_threshold, p.d_key_in);
        sort_in = p.d_key_in;
        lo_bit = 0;
        hi_bit = 29;
    }
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, sort_in, p.d_keys, p.d_iota,
                                              p.d_order, a.n, lo_bit, hi_bit, stream);
    FPH_CUDA_TRY(cudaMallocAsync(&p.tmp, tmp_bytes, stream));
    FPH_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(p.tmp, tmp_bytes, sort_in, p.d_keys,
                                                           p.d_iota, p.d_order, a.n, lo_bit,
                                                           hi_bit, stream));
    while (p.nk < 4 && p.kern[p.nk]) ++p.nk;
    FPH_CUDA_TRY(cudaMallocAsync(&p.d_counters, sizeof(int) * 4, stream));
    FPH_CUDA_TRY(cudaMemsetAsync(p.d_counters, 0, sizeof(int) * 4, stream));
    if (p.nk > 1) {
        FPH_CUDA_TRY(cudaMallocAsync(&p.d_stage, sizeof(int) * a.n, stream));
        FPH_CUDA_TRY(cudaMemsetAsync(p.d_stage, 0, sizeof(int) * a.n, stream));
    }
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

int search_run(SearchPlan& p, bool release) {
    for (int i = 0; i < p.nk; ++i) {
        FPH_CUDA_TRY(cudaFuncSetAttribute(p.kern[i], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          p.smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.blocks);
        cfg.blockDim = dim3(kSThreads);
        cfg.dynamicSmemBytes = p.smem;
        cfg.stream = p.stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        // PDL between the chain's phases (per-simplex stage flags order them)
        cfg.numAttrs = (i > 0 && p.d_stage) ? 1 : 0;
        FPH_CUDA_TRY(cudaLaunchKernelEx(&cfg, p.kern[i], p.b, p.d_geom, (const int*)p.d_order,
                                        p.d_counters + i, p.d_stage, i));
    }
    FPH_CUDA_TRY(cudaGetLastError());
    return release ? search_release(p) : FPH_OK;
}

int search_release(SearchPlan& p) {
    for (void* q : {(void*)p.d_counters, (void*)p.d_stage, (void*)p.d_lower, (void*)p.d_thr,
                    (void*)p.d_keys, (void*)p.d_order, (void*)p.d_iota, p.tmp, (void*)p.d_key_in})
        if (q) FPH_CUDA_TRY(cudaFreeAsync(q, p.stream));
    p = SearchPlan{};
    return FPH_OK;
}

int launch_search(const FloodArgs& a, const SimplexGeom* d_geom, const int* d_cand,
                  cudaStream_t stream) {
    SearchPlan p;
    FPH_TRY(search_prepare(a, d_geom, d_cand, stream, &p));
    return search_run(p, true);
}

}  // namespace FPH_SLOT_NS

}  // namespace fph
