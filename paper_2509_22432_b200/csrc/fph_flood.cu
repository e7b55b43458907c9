// fph_flood.cu -- the flooding kernel: per-simplex max over barycentric
// sample points of the min distance to the cloud.
//
// Replaces the reference's masked minimisation (floodph/filtration.py:233
// _grid_values_masked, :130 compute_mask, floodph/_kernels.py:41
// _min_sq_dists_nb).  The reference values every grid row of each top cell
// against the cloud points inside the cell's sqrt(2)-inflated Ritter ball
// and reads face values off the cell's grid.  Because face rows are bitwise
// the face's own grid rows (reference test_geometry.py
// test_grid_face_rows_bitwise_equal_own_grid) and max is exact, the value of
// a simplex equals max(value over its RELATIVE-INTERIOR rows, values of its
// facets); this file computes the interior part once per simplex of every
// dimension (no row is evaluated twice) and fph_complete_kernel folds in the
// facets.
//
// Numerics.  Results are bit-identical to the reference's float64 values:
//   1. fp32 pass: sample point b and candidates a are taken relative to the
//      simplex's Ritter center (float64 subtract, one rounding to fp32), and
//      q = |a|^2 - 2 a.b is evaluated with packed FFMA2 (two candidates per
//      instruction) and a 3-input FMNMX3 -- 3 FFMA2 + 1 FMNMX3 per 2 pairs.
//      m32(p) = min q + |b|^2 differs from the exact squared distance by at
//      most E(p) = 40 u32 (|b| + sqrt(m32))^2 (derivation in DESIGN.md).
//   2. exact refine: only points with m32 + E >= max_p (m32 - E) can hold
//      the maximum; each is re-evaluated in float64 with the reference's
//      operation order over the grid cells of the small ball
//      |x - p| <= sqrt(m32 + 2E), which provably contains the float64
//      nearest neighbour.  The max of those exact minima is the reference's
//      value.  Points are visited in decreasing m32 and skipped once they
//      cannot beat the running max, so usually 1-3 points are refined.
#include <cub/cub.cuh>

#include <cfloat>
#include <cmath>
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "fph_dev.cuh"
#include "fph_flood.cuh"

namespace fph {

namespace {

constexpr int kThreads = 256;
constexpr int kTile = 2048;           // candidates staged per flush (32 KB)

// work counters (profiling aid, read by fph_flood_stats):
// 0 fp32 pairs evaluated, 1 candidates staged, 2 candidates scanned,
// 3 refined points, 4 float64 refine distances, 5 tasks
// block search: 7 blocks, 8 blocks pruned whole, 9 points certified in
// round 1, 10 points needing more after round 1, 11 representative passes,
// 12 round-2 passes, 13/14/15 candidates scanned in round 1 / reps (incl.
// counting) / round 2, 16/17/18 staged in round 1 / reps / round 2
constexpr int kStats = 24;
__device__ unsigned long long g_stats[kStats];

// ------------------------------------------------------------ block scan
// exclusive prefix sum over the CTA; returns the total in `total`
__device__ __forceinline__ int block_excl(int v, int* warp_buf, int& total) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) warp_buf[w] = incl;
    __syncthreads();
    if (w == 0) {
        int x = lane < (kThreads / 32) ? warp_buf[lane] : 0;
        int xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < (kThreads / 32)) warp_buf[lane] = xi - x;
        if (lane == (kThreads / 32) - 1) warp_buf[kThreads / 32] = xi;
    }
    __syncthreads();
    total = warp_buf[kThreads / 32];
    return warp_buf[w] + incl - v;
}

__device__ __forceinline__ float block_max_f(float v, float* buf) {
    v = warp_max(v);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) buf[w] = v;
    __syncthreads();
    float r = buf[0];
    for (int i = 1; i < kThreads / 32; ++i) r = fmaxf(r, buf[i]);
    __syncthreads();
    return r;
}

__device__ __forceinline__ double block_min_d(double v, double* buf) {
    v = warp_min_d(v);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) buf[w] = v;
    __syncthreads();
    double r = buf[0];
    for (int i = 1; i < kThreads / 32; ++i) r = fmin(r, buf[i]);
    __syncthreads();
    return r;
}

// ------------------------------------------------------------ setup
// One warp per simplex: Ritter ball, candidate cell box, candidate count,
// and the number of tasks the simplex is split into.
__global__ void setup_kernel(FloodArgs a, SimplexGeom* __restrict__ geom,
                             int* __restrict__ ntasks) {
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= a.n) return;
    const Grid g = *a.gp;
    Verts V;
    load_verts(a, warp, V);
    SimplexGeom G;
    double c[3];
    double r = ritter(V, a.k, c);
    G.cx = c[0];
    G.cy = c[1];
    G.cz = c[2];
    G.r = r;
    // sqrt(2) r: Lemma 4.2 masking radius; tiny relative slack for rounding
    G.rho = a.subset ? 1.4142135623730951 * r * (1.0 + 1e-9) : 0.0;
    Box b = a.subset ? ball_box(g, c[0], c[1], c[2], G.rho) : full_box(g);
    G.box = b;
    int rows = b.rows();
    long long cand = 0;
    if (a.nblk > 0) {
        // bounded search: the count only steers sampling and scheduling, so
        // an estimate suffices -- fp32 row clipping, every `step`-th row,
        // about 256 rows of a large ball (a hull simplex of box_10m spans
        // ~10^5 grid rows; every 4th of them made this kernel 0.14 ms)
#ifndef FPH_SETUP_ROWS
#define FPH_SETUP_ROWS 256
#endif
        const int step = (FPH_SETUP_ROWS > 0 && rows > 4 * FPH_SETUP_ROWS)
                             ? ((rows / FPH_SETUP_ROWS) | 1)
                             : (rows > 512 ? 4 : (rows > 128 ? 2 : 1));
        const RowClipF cf = make_clip_f(g, c[0], c[1], c[2], G.rho);
#pragma unroll 4
        for (int rr = lane * step; rr < rows; rr += 32 * step) {
            int2 run;
            if (a.subset) {
                run = row_run_f(g, b, rr, cf);
            } else {
                const int base = ((b.z0 + rr / b.ny_b()) * g.ny + b.y0 + rr % b.ny_b()) * g.nx;
                run = make_int2(g.cell_start[base + b.x0], g.cell_start[base + b.x1 + 1]);
            }
            cand += (long long)(run.y - run.x) * step;
        }
    } else {
        for (int rr = lane; rr < rows; rr += 32) {
            int2 run = row_run(g, b, rr, c[0], c[1], c[2], G.rho, a.subset != 0);
            cand += run.y - run.x;
        }
    }
    for (int o = 16; o > 0; o >>= 1) cand += __shfl_xor_sync(0xffffffffu, cand, o);
    int npc = (a.P + a.chunk_pts - 1) / a.chunk_pts;
    int pc = min(a.P, a.chunk_pts);
    double pairs = (double)pc * (double)cand;
    int nrp = (int)fmin(fmax(1.0, ceil(pairs / a.pairs_per_task)), (double)max(rows, 1));
    G.nrp = nrp;
    G.npc = npc;
    if (lane == 0) {
        geom[warp] = G;
        ntasks[warp] = a.P > 0 ? npc * nrp : 0;
        if (a.cand_count) a.cand_count[warp] = (int)min(cand, (long long)0x7fffffff);
    }
}

// --------------------------------------------------------- fp32 pass
struct SmemPass {
    float4 tileA[kTile / 2];  // pair p: (c0.x, c1.x, c0.y, c1.y)
    float4 tileB[kTile / 2];  //         (c0.z, c1.z, c0.w, c1.w)
    int row_off[kThreads + 1];
    int row_beg[kThreads];
    int warp_buf[kThreads / 32 + 1];
    float fbuf[kThreads / 32];
    double dbuf[kThreads / 32];
    int task, last;
    int list[kThreads];
    int list_n;
};

template <int PPT>
__device__ __forceinline__ void compute_tile(SmemPass& S, int n, int g, int G, bool active,
                                             const float (&bx)[PPT], const float (&by)[PPT],
                                             const float (&bz)[PPT], float (&best)[PPT]) {
    if ((n & 1) && threadIdx.x == 0) {
        float* A = reinterpret_cast<float*>(S.tileA);
        float* B = reinterpret_cast<float*>(S.tileB);
        int p = n >> 1;
        A[p * 4 + 1] = 0.f;
        A[p * 4 + 3] = 0.f;
        B[p * 4 + 1] = 0.f;
        B[p * 4 + 3] = INFINITY;  // w = +inf: never the minimum
    }
    __syncthreads();
    if (active) {
        int np = (n + 1) >> 1;
        int p0 = (int)((long long)np * g / G), p1 = (int)((long long)np * (g + 1) / G);
#pragma unroll 2
        for (int p = p0; p < p1; ++p) {
            float4 A = S.tileA[p];
            float4 B = S.tileB[p];
            float2 cx = make_float2(A.x, A.y), cy = make_float2(A.z, A.w);
            float2 cz = make_float2(B.x, B.y), cw = make_float2(B.z, B.w);
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                float2 acc = ffma2(make_float2(bz[i], bz[i]), cz, cw);
                acc = ffma2(make_float2(by[i], by[i]), cy, acc);
                acc = ffma2(make_float2(bx[i], bx[i]), cx, acc);
                best[i] = fmin3(best[i], acc.x, acc.y);
            }
        }
    }
    __syncthreads();
}

// Exact float64 nearest-neighbour squared distance of p over the grid cells
// of the ball |x - p| <= R (cooperative over the CTA).
__device__ __noinline__ double refine_point(const Grid& g, SmemPass& S, const double p[3], double R) {
    Box b = ball_box(g, p[0], p[1], p[2], R);
    int rows = b.rows();
    double best = INFINITY;
    unsigned long long scanned = 0;
    for (int rb = 0; rb < rows; rb += kThreads) {
        int r = rb + threadIdx.x;
        int2 run = r < rows ? row_run(g, b, r, p[0], p[1], p[2], R, true) : make_int2(0, 0);
        int total;
        int off = block_excl(run.y - run.x, S.warp_buf, total);
        S.row_off[threadIdx.x] = off;
        S.row_beg[threadIdx.x] = run.x;
        __syncthreads();
        int nrow = min(kThreads, rows - rb);
        scanned += total;
        for (int f = threadIdx.x; f < total; f += kThreads) {
            int lo = 0, hi = nrow;  // last row with off <= f
            while (hi - lo > 1) {
                int mid = (lo + hi) >> 1;
                if (S.row_off[mid] <= f) lo = mid; else hi = mid;
            }
            int idx = S.row_beg[lo] + f - S.row_off[lo];
            best = fmin(best, sq64(g.x[idx], g.y[idx], g.z[idx], p[0], p[1], p[2]));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        atomicAdd(&g_stats[3], 1ull);
        atomicAdd(&g_stats[4], scanned);
    }
    return block_min_d(best, S.dbuf);
}

// |b| (fp32) of point j, recomputed: the Ritter center is per simplex
__device__ __forceinline__ float point_b(const FloodArgs& a, const Verts& V, const SimplexGeom& G,
                                         int s, int j) {
    double p[3];
    sample_row(a, V, s, j, nullptr, p);
    float fx = __double2float_rn(__dsub_rn(p[0], G.cx));
    float fy = __double2float_rn(__dsub_rn(p[1], G.cy));
    float fz = __double2float_rn(__dsub_rn(p[2], G.cz));
    return sqrtf(fmaf(fz, fz, fmaf(fy, fy, fx * fx))) * 1.0001f;
}

// Finalize one simplex: pick the refine set from the fp32 minima and
// return the exact float64 max over it.
__device__ __noinline__ double finalize(const FloodArgs& a, SmemPass& S, int s, const Verts& V,
                           const SimplexGeom& G) {
    const float* m32 = a.perpoint + (size_t)s * a.P;
    // L = max_p (m32 - E), and the argmax of m32
    double lmax = -INFINITY;
    float vmax = -INFINITY;
    int jmax = 0x7fffffff;
    for (int j = threadIdx.x; j < a.P; j += kThreads) {
        float v = __ldcg(m32 + j);
        float B = point_b(a, V, G, s, j);
        float sv = sqrtf(fmaxf(v, 0.f)) + B;
        float E = (float)(40.0 * kU32 * 1.01) * sv * sv;
        lmax = fmax(lmax, (double)v - (double)E);
        if (v > vmax) {
            vmax = v;
            jmax = j;
        }
    }
    double L = -block_min_d(-lmax, S.dbuf);
    // argmax (lowest index among ties; any maximiser works)
    float vm = block_max_f(vmax, S.fbuf);
    int cand = vmax == vm ? jmax : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
    if ((threadIdx.x & 31) == 0) S.row_beg[threadIdx.x >> 5] = cand;
    __syncthreads();
    int jm = S.row_beg[0];
    for (int w = 1; w < kThreads / 32; ++w) jm = min(jm, S.row_beg[w]);
    __syncthreads();

    double M = -INFINITY;
    // refine the fp32 argmax first, then anything that can still beat M
    for (int pass = 0; pass < 2; ++pass) {
        for (int base = 0; base < (pass == 0 ? 1 : a.P); base += kThreads) {
            int j = pass == 0 ? jm : base + threadIdx.x;
            bool want = false;
            float v = 0.f, E = 0.f;
            if ((pass == 0 && threadIdx.x == 0) || (pass == 1 && j < a.P && j != jm)) {
                v = __ldcg(m32 + j);
                float B = point_b(a, V, G, s, j);
                float sv = sqrtf(fmaxf(v, 0.f)) + B;
                E = (float)(40.0 * kU32 * 1.01) * sv * sv;
                want = (double)v + (double)E >= (double)L && (double)v + (double)E > M;
            }
            int tot;
            int pos = block_excl(want ? 1 : 0, S.warp_buf, tot);
            if (want) S.list[pos] = j;
            __syncthreads();
            for (int t = 0; t < tot; ++t) {
                int jj = S.list[t];
                float vv = __ldcg(m32 + jj);
                float B = point_b(a, V, G, s, jj);
                float sv = sqrtf(fmaxf(vv, 0.f)) + B;
                float EE = (float)(40.0 * kU32 * 1.01) * sv * sv;
                if ((double)vv + (double)EE <= M) continue;  // uniform across the CTA
                double p[3];
                sample_row(a, V, s, jj, nullptr, p);
                double R2 = fmax((double)vv + 2.0 * (double)EE, 0.0);
                double R = sqrt(R2) * (1.0 + 1e-6) + 1e-300;
                double m64 = refine_point(*a.gp, S, p, R);
                M = fmax(M, m64);
            }
            __syncthreads();
        }
    }
    return M;
}

template <int PPT>
__global__ void __launch_bounds__(kThreads, 2) pass_kernel(FloodArgs a, const SimplexGeom* geom,
                                                        const int* task_off, int* task_counter,
                                                        int* done) {
    __shared__ SmemPass S;
    const Grid grid = *a.gp;
    const int total_tasks = task_off[a.n];
    for (;;) {
        if (threadIdx.x == 0) S.task = atomicAdd(task_counter, 1);
        __syncthreads();
        const int t = S.task;
        __syncthreads();
        if (t >= total_tasks) return;
        // simplex owning task t: last s with task_off[s] <= t
        int lo = 0, hi = a.n;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (task_off[mid] <= t) lo = mid; else hi = mid;
        }
        const int s = lo;
        const SimplexGeom G = geom[s];
        const int jt = t - task_off[s];
        const int nt = G.npc * G.nrp;
        const int pc = jt % G.npc, rp = jt / G.npc;
        const int rows = G.box.rows();
        const int row_lo = (int)((long long)rows * rp / G.nrp);
        const int row_hi = (int)((long long)rows * (rp + 1) / G.nrp);
        const int pbase = pc * a.chunk_pts;
        const int Pc = min(a.P - pbase, a.chunk_pts);
        const int Q = (Pc + PPT - 1) / PPT;
        const int Gn = kThreads / Q;
        const int slot = threadIdx.x % Q, g = threadIdx.x / Q;
        const bool active = g < Gn;
        Verts V;
        load_verts(a, s, V);
        float bx[PPT], by[PPT], bz[PPT], bb[PPT], best[PPT];
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            int jl = min(slot * PPT + i, Pc - 1);
            double p[3];
            sample_row(a, V, s, pbase + jl, nullptr, p);
            float fx = __double2float_rn(__dsub_rn(p[0], G.cx));
            float fy = __double2float_rn(__dsub_rn(p[1], G.cy));
            float fz = __double2float_rn(__dsub_rn(p[2], G.cz));
            bx[i] = -2.f * fx;
            by[i] = -2.f * fy;
            bz[i] = -2.f * fz;
            bb[i] = fmaf(fz, fz, fmaf(fy, fy, fx * fx));
            best[i] = INFINITY;
        }
        const float thr = a.subset ? (float)(G.rho * G.rho * (1.0 + 1e-5)) : INFINITY;
        int tile_n = 0;
        unsigned long long n_staged = 0, n_scanned = 0;
        for (int rb = row_lo; rb < row_hi; rb += kThreads) {
            int r = rb + threadIdx.x;
            int2 run = r < row_hi ? row_run(grid, G.box, r, G.cx, G.cy, G.cz, G.rho, a.subset != 0)
                                  : make_int2(0, 0);
            int total;
            int off = block_excl(run.y - run.x, S.warp_buf, total);
            S.row_off[threadIdx.x] = off;
            S.row_beg[threadIdx.x] = run.x;
            __syncthreads();
            const int nrow = min(kThreads, row_hi - rb);
            n_scanned += total;
            for (int f0 = 0; f0 < total; f0 += kThreads) {
                int f = f0 + (int)threadIdx.x;
                bool keep = false;
                float ax = 0.f, ay = 0.f, az = 0.f, aw = 0.f;
                if (f < total) {
                    int l = 0, h = nrow;
                    while (h - l > 1) {
                        int mid = (l + h) >> 1;
                        if (S.row_off[mid] <= f) l = mid; else h = mid;
                    }
                    int idx = S.row_beg[l] + f - S.row_off[l];
                    ax = __double2float_rn(__dsub_rn(grid.x[idx], G.cx));
                    ay = __double2float_rn(__dsub_rn(grid.y[idx], G.cy));
                    az = __double2float_rn(__dsub_rn(grid.z[idx], G.cz));
                    aw = fmaf(az, az, fmaf(ay, ay, ax * ax));
                    keep = aw <= thr;
                }
                int kept;
                int pos = block_excl(keep ? 1 : 0, S.warp_buf, kept);
                if (keep) {
                    int q = tile_n + pos;
                    float* A = reinterpret_cast<float*>(S.tileA) + (q >> 1) * 4 + (q & 1);
                    float* B = reinterpret_cast<float*>(S.tileB) + (q >> 1) * 4 + (q & 1);
                    A[0] = ax;
                    A[2] = ay;
                    B[0] = az;
                    B[2] = aw;
                }
                tile_n += kept;
                n_staged += kept;
                if (tile_n > kTile - kThreads) {
                    compute_tile<PPT>(S, tile_n, g, Gn, active, bx, by, bz, best);
                    tile_n = 0;
                }
            }
            __syncthreads();
        }
        if (tile_n > 0) compute_tile<PPT>(S, tile_n, g, Gn, active, bx, by, bz, best);
        if (threadIdx.x == 0) {
            atomicAdd(&g_stats[0], n_staged * (unsigned long long)Pc);
            atomicAdd(&g_stats[1], n_staged);
            atomicAdd(&g_stats[2], n_scanned);
            atomicAdd(&g_stats[5], 1ull);
        }
        // reduce the groups' partial minima: red[g][jl], reusing the tile
        float* red = reinterpret_cast<float*>(S.tileA);
        if (active) {
#pragma unroll
            for (int i = 0; i < PPT; ++i) red[g * (Q * PPT) + slot * PPT + i] = best[i] + bb[i];
        }
        __syncthreads();
        float* out = a.perpoint + (size_t)s * a.P + pbase;
        for (int jl = threadIdx.x; jl < Pc; jl += kThreads) {
            float v = red[jl];
            for (int gg = 1; gg < Gn; ++gg) v = fminf(v, red[gg * (Q * PPT) + jl]);
            if (nt == 1) out[jl] = v;
            else atomicMin(reinterpret_cast<unsigned*>(out) + jl, f2ord(v));
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) S.last = nt == 1 ? 1 : (atomicAdd(done + s, 1) == nt - 1);
        __syncthreads();
        if (!S.last) continue;
        __threadfence();
        if (nt > 1) {  // decode the ordered-uint minima in place
            for (int j = threadIdx.x; j < a.P; j += kThreads) {
                unsigned* u = reinterpret_cast<unsigned*>(a.perpoint + (size_t)s * a.P) + j;
                *u = __float_as_uint(ord2f(__ldcg(u)));
            }
            __threadfence();
            __syncthreads();
        }
        double M = finalize(a, S, s, V, G);
        if (threadIdx.x == 0) a.out_sq[s] = M;
        __syncthreads();
    }
}


__global__ void init_perpoint_kernel(unsigned* p, long long n) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) p[i] = 0xffffffffu;
}

__global__ void no_interior_kernel(double* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = -1.0;
}

}  // namespace

int choose_ppt(int P) {
    // Issue-slot model of the inner loop: per candidate pair a thread issues
    // 2 LDS.128 + PPT x (3 FFMA2 + 1 FMNMX3); the G = kThreads / Q groups of
    // a task (Q = ceil(pc / PPT) threads each) split the tile.  Minimise the
    // summed per-pair cost over all point chunks.  Groups narrower than 4
    // threads would scatter a warp's tile reads over too many addresses.
    int best = 1;
    double best_cost = 1e300;
    for (int ppt : {1, 2, 4, 8}) {
        const int chunk = kThreads * ppt;
        double cost = 0.0;
        bool ok = true;
        for (int base = 0; base < P; base += chunk) {
            int pc = P - base < chunk ? P - base : chunk;
            int Q = (pc + ppt - 1) / ppt;
            if (Q < 4 && ppt > 1) ok = false;
            cost += (2.0 + 4.0 * ppt) / (kThreads / Q);
        }
        if (ok && cost < best_cost - 1e-12) {
            best_cost = cost;
            best = ppt;
        }
    }
    return best;
}

// ---------------------------------------------------------- profiling
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_pass_events, g_grid_events;
static double g_pass_ms = 0.0, g_grid_ms = 0.0;

void profile_push(cudaEvent_t a, cudaEvent_t b) { g_pass_events.emplace_back(a, b); }
void profile_push_grid(cudaEvent_t a, cudaEvent_t b) { g_grid_events.emplace_back(a, b); }

int flood_stats(double* out, int reset) {
    for (auto& e : g_pass_events) {
        FPH_CUDA_TRY(cudaEventSynchronize(e.second));
        float ms = 0.f;
        FPH_CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
        g_pass_ms += ms;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    g_pass_events.clear();
    for (auto& e : g_grid_events) {
        FPH_CUDA_TRY(cudaEventSynchronize(e.second));
        float ms = 0.f;
        FPH_CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
        g_grid_ms += ms;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    g_grid_events.clear();
    unsigned long long h[kStats];
    FPH_CUDA_TRY(cudaMemcpyFromSymbol(h, g_stats, sizeof(h)));
    for (int i = 0; i < kStats; ++i) out[i] = (double)h[i];
    out[6] = g_pass_ms;
    out[23] = g_grid_ms;
    if (reset) {
        unsigned long long z[kStats] = {};
        FPH_CUDA_TRY(cudaMemcpyToSymbol(g_stats, z, sizeof(z)));
        g_pass_ms = 0.0;
        g_grid_ms = 0.0;
    }
    return FPH_OK;
}

// Debug capture (profiling aid): per flood_range launch with the search
// kernels, kDbgFields values per simplex (search_kernel fills them); the
// device buffers are kept until debug_fetch, which waits for the device and
// returns blocks [k, n, n x kDbgFields values] -- no stream sync in between,
// so the captured run keeps its concurrency.
struct DebugRec {
    long long* d;
    int n, k;
};
static bool g_debug = false;
static std::vector<DebugRec> g_debug_pending;
static std::vector<long long> g_debug_buf;
void debug_enable(bool on) {
    g_debug = on;
    if (on) g_debug_buf.clear();
}
int debug_fetch(long long* out, long long cap, long long* n) {
    if (!g_debug_pending.empty()) {
        FPH_CUDA_TRY(cudaDeviceSynchronize());
        for (const DebugRec& r : g_debug_pending) {
            const size_t base = g_debug_buf.size();
            g_debug_buf.resize(base + 2 + (size_t)kDbgFields * r.n);
            g_debug_buf[base] = r.k;
            g_debug_buf[base + 1] = r.n;
            FPH_CUDA_TRY(cudaMemcpy(g_debug_buf.data() + base + 2, r.d,
                                    sizeof(long long) * kDbgFields * r.n, cudaMemcpyDeviceToHost));
            FPH_CUDA_TRY(cudaFree(r.d));
        }
        g_debug_pending.clear();
    }
    *n = (long long)g_debug_buf.size();
    if (out) std::copy(g_debug_buf.begin(), g_debug_buf.begin() + std::min<long long>(cap, *n), out);
    return FPH_OK;
}

namespace {

// Row templates per (device, k, m) -- or per explicit row count -- built on
// the host once and kept on the device: the compositions of m into k + 1
// positive parts (k = 0: the vertex) grouped into lattice tiles of <= 32 rows
// (t^k rows, t = 32, 5, 3 for k = 1, 2, 3) and ordered center-first: blocks
// near the barycenter tend to hold the maximum, which raises the shared
// lower bound early.  Explicit rows (uniform-random sampler) are blocks of 32
// consecutive samples.
struct Template {
    ushort4* rows = nullptr;  // P rows
    int* blk_off = nullptr;   // nblk + 1
    int P = 0, nblk = 0;
};

std::mutex g_tmpl_mu;
std::map<std::tuple<int, int, int, int>, Template> g_tmpl;

int build_template(int k, int m, int explicit_rows, Template* out) {
    std::vector<ushort4> rows;
    std::vector<int> blk_off;
    if (explicit_rows > 0) {
        rows.assign(explicit_rows, make_ushort4(0, 0, 0, 0));
        for (int b = 0; b < explicit_rows; b += 32) blk_off.push_back(b);
    } else {
        std::vector<ushort4> all;
        auto u = [](int v) { return (unsigned short)v; };
        if (k == 0) {
            all.push_back(make_ushort4(u(m), 0, 0, 0));
        } else if (k == 1) {
            for (int c0 = 1; c0 <= m - 1; ++c0) all.push_back(make_ushort4(u(c0), u(m - c0), 0, 0));
        } else if (k == 2) {
            for (int c0 = 1; c0 <= m - 2; ++c0)
                for (int c1 = 1; c1 <= m - 1 - c0; ++c1)
                    all.push_back(make_ushort4(u(c0), u(c1), u(m - c0 - c1), 0));
        } else {
            for (int c0 = 1; c0 <= m - 3; ++c0)
                for (int c1 = 1; c1 <= m - 2 - c0; ++c1)
                    for (int c2 = 1; c2 <= m - 1 - c0 - c1; ++c2)
                        all.push_back(make_ushort4(u(c0), u(c1), u(c2), u(m - c0 - c1 - c2)));
        }
        const int tile = k <= 1 ? 32 : (k == 2 ? 5 : 3);
        std::vector<std::pair<long long, int>> keyed;  // (tile key, row)
        keyed.reserve(all.size());
        for (int i = 0; i < (int)all.size(); ++i) {
            const ushort4 c = all[i];
            const long long key = k <= 1 ? (c.x - 1) / tile
                                         : ((long long)(c.x / tile) * 65536 + c.y / tile) * 65536 +
                                               (k == 3 ? c.z / tile : 0);
            keyed.emplace_back(key, i);
        }
        std::stable_sort(keyed.begin(), keyed.end(),
                         [](const std::pair<long long, int>& x, const std::pair<long long, int>& y) {
                             return x.first < y.first;
                         });
        struct Blk { double dist; int beg, end; };
        std::vector<Blk> blks;
        for (int i = 0; i < (int)keyed.size();) {
            int j = i;
            double mc[4] = {0, 0, 0, 0};
            while (j < (int)keyed.size() && keyed[j].first == keyed[i].first) {
                const ushort4 c = all[keyed[j].second];
                mc[0] += c.x; mc[1] += c.y; mc[2] += c.z; mc[3] += c.w;
                ++j;
            }
            double d = 0.0;
            for (int t = 0; t <= k; ++t) {
                const double e = mc[t] / (j - i) / m - 1.0 / (k + 1);
                d += e * e;
            }
            blks.push_back({d, i, j});
            i = j;
        }
        std::stable_sort(blks.begin(), blks.end(),
                         [](const Blk& x, const Blk& y) { return x.dist < y.dist; });
        rows.reserve(all.size());
        for (const Blk& bk : blks) {
            blk_off.push_back((int)rows.size());
            for (int i = bk.beg; i < bk.end; ++i) rows.push_back(all[keyed[i].second]);
        }
    }
    blk_off.push_back((int)rows.size());
    Template t;
    t.P = (int)rows.size();
    t.nblk = (int)blk_off.size() - 1;
    if (t.P > 0) {
        FPH_CUDA_TRY(cudaMalloc(&t.rows, sizeof(ushort4) * t.P));
        FPH_CUDA_TRY(cudaMemcpy(t.rows, rows.data(), sizeof(ushort4) * t.P, cudaMemcpyHostToDevice));
    }
    FPH_CUDA_TRY(cudaMalloc(&t.blk_off, sizeof(int) * blk_off.size()));
    FPH_CUDA_TRY(cudaMemcpy(t.blk_off, blk_off.data(), sizeof(int) * blk_off.size(),
                            cudaMemcpyHostToDevice));
    *out = t;
    return FPH_OK;
}

int get_template(int k, int m, int explicit_rows, Template* out) {
    int dev = 0;
    FPH_CUDA_TRY(cudaGetDevice(&dev));
    const auto key = std::make_tuple(dev, k, explicit_rows > 0 ? 0 : m, explicit_rows);
    std::lock_guard<std::mutex> lock(g_tmpl_mu);
    auto it = g_tmpl.find(key);
    if (it == g_tmpl.end()) {
        Template t;
        FPH_TRY(build_template(k, m, explicit_rows, &t));
        it = g_tmpl.emplace(key, t).first;
    }
    *out = it->second;
    return FPH_OK;
}

// Interior rows of a k-simplex at resolution m: C(m - 1, k).
long long interior_rows(int k, int m) {
    if (k == 0) return 1;
    long long r = 1;
    for (int i = 0; i < k; ++i) r = r * (m - 1 - i) / (i + 1);
    return m - 1 >= k ? r : 0;
}

// per-point fp32 scratch per chunk of simplices (n x P floats)
constexpr double kPerpointBudget = 2.0 * (1 << 30);

// One chunk of simplices of one dimension, queued in two steps
// (range_prepare: allocations, setup_kernel, the search set-up; range_run:
// the flooding kernels and the frees).
struct RangePlan {
    FloodArgs a{};
    bool search = false, profile = false;
    int ppt = 1;
    int slot = 0;  // the search kernels' grid slot (FloodTuning::grid_slot)
    cudaStream_t stream = nullptr;
    SimplexGeom* d_geom = nullptr;
    int *d_ntasks = nullptr, *d_task_off = nullptr, *d_counter = nullptr, *d_done = nullptr;
    int* d_cand = nullptr;
    float* d_perpoint = nullptr;
    void* tmp = nullptr;
    SearchPlan sp;
};

int range_prepare(const Grid* d_grid, const double* d_landmarks3, const int* d_simplices, int n,
                  int k, int m, int subset, double* d_out_sq, const FloodTuning& tune,
                  cudaStream_t stream, const double* d_explicit, const Template& T,
                  RangePlan* plan) {
    RangePlan& rp = *plan;
    rp = RangePlan{};
    rp.stream = stream;
    rp.profile = tune.profile;
    const int P = T.P;
    rp.ppt = choose_ppt(P);
    FloodArgs& a = rp.a;
    a.gp = d_grid;
    a.landmarks = d_landmarks3;
    a.simplices = d_simplices;
    a.n = n;
    a.k = k;
    a.m = m;
    a.P = P;
    a.subset = subset;
    a.chunk_pts = kThreads * rp.ppt;
    a.pairs_per_task = tune.pairs_per_task > 0 ? tune.pairs_per_task : (double)(1 << 21);
    a.out_sq = d_out_sq;
    a.explicit_pts = d_explicit;
    // the bounded search keeps the (m + 1) weights in shared memory; a
    // resolution too large for that takes the brute-force kernel
    const int gslot = tune.grid_slot;
    const size_t sbytes = gslot == 2 ? slot2::search_smem_bytes(P, m)
                                     : slot0::search_smem_bytes(P, m);  // slots 0, 1: one build
    const size_t slimit = gslot == 2 ? slot2::search_smem_limit() : slot0::search_smem_limit();
    rp.search = tune.algo >= 1 && sbytes <= slimit;
    a.nblk = rp.search ? T.nblk : 0;
    a.reps_target = tune.reps_target > 0 ? tune.reps_target : 384;
    a.team_threshold = tune.team_threshold;
    a.team_thr_dev = nullptr;
    a.exact_pairs = tune.exact_pairs;
    for (int i = 0; i < 4; ++i) a.exact_cand[i] = tune.exact_cand[i];
    a.points_per_landmark = tune.points_per_landmark;
    a.tmpl = T.rows;
    a.blk_off = T.blk_off;

    FPH_CUDA_TRY(cudaMallocAsync(&rp.d_geom, sizeof(SimplexGeom) * n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&rp.d_ntasks, sizeof(int) * (n + 1), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&rp.d_task_off, sizeof(int) * (n + 1), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&rp.d_counter, sizeof(int), stream));
    FPH_CUDA_TRY(cudaMallocAsync(&rp.d_done, sizeof(int) * n, stream));
    FPH_CUDA_TRY(cudaMallocAsync(&rp.d_perpoint, sizeof(float) * (size_t)n * P, stream));
    FPH_CUDA_TRY(cudaMemsetAsync(rp.d_counter, 0, sizeof(int), stream));
    FPH_CUDA_TRY(cudaMemsetAsync(rp.d_done, 0, sizeof(int) * n, stream));
    FPH_CUDA_TRY(cudaMemsetAsync(rp.d_ntasks + n, 0, sizeof(int), stream));
    const long long npp = (long long)n * P;
    if (!rp.search)
        init_perpoint_kernel<<<(unsigned)((npp + 255) / 256), 256, 0, stream>>>(
            reinterpret_cast<unsigned*>(rp.d_perpoint), npp);
    if (rp.search) FPH_CUDA_TRY(cudaMallocAsync(&rp.d_cand, sizeof(int) * n, stream));
    a.cand_count = rp.d_cand;
    FPH_CUDA_TRY(cudaGetSymbolAddress((void**)&a.stats, g_stats));
    a.perpoint = rp.d_perpoint;

    setup_kernel<<<(n * 32 + 255) / 256, 256, 0, stream>>>(a, rp.d_geom, rp.d_ntasks);
    if (!rp.search) {
        size_t tmp_bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rp.d_ntasks, rp.d_task_off, n + 1, stream);
        FPH_CUDA_TRY(cudaMallocAsync(&rp.tmp, tmp_bytes, stream));
        FPH_CUDA_TRY(cub::DeviceScan::ExclusiveSum(rp.tmp, tmp_bytes, rp.d_ntasks, rp.d_task_off,
                                                   n + 1, stream));
    }
    long long* d_dbg = nullptr;
    if (rp.search && g_debug) {
        // stream-ordered: a plain cudaMalloc here could wait for the device
        // and serialise the dimensions of the captured run
        FPH_CUDA_TRY(cudaMallocAsync(&d_dbg, sizeof(long long) * kDbgFields * n, stream));
        FPH_CUDA_TRY(cudaMemsetAsync(d_dbg, 0, sizeof(long long) * kDbgFields * n, stream));
        g_debug_pending.push_back({d_dbg, n, k});
    }
    a.dbg = d_dbg;
    rp.slot = tune.grid_slot;
    if (rp.search)
        FPH_TRY(rp.slot == 2   ? slot2::search_prepare(a, rp.d_geom, a.cand_count, stream, &rp.sp)
                : rp.slot == 1 ? slot1::search_prepare(a, rp.d_geom, a.cand_count, stream, &rp.sp)
                               : slot0::search_prepare(a, rp.d_geom, a.cand_count, stream, &rp.sp));
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

int range_run(RangePlan& rp) {
    cudaStream_t stream = rp.stream;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (rp.profile) {
        FPH_CUDA_TRY(cudaEventCreate(&ev0));
        FPH_CUDA_TRY(cudaEventCreate(&ev1));
        FPH_CUDA_TRY(cudaEventRecord(ev0, stream));
    }
    if (rp.search) {
        FPH_TRY(rp.slot == 2   ? slot2::search_run(rp.sp, true)
                : rp.slot == 1 ? slot1::search_run(rp.sp, true)
                               : slot0::search_run(rp.sp, true));
    } else {
        int dev = 0, sms = 0, occ = 0;
        FPH_CUDA_TRY(cudaGetDevice(&dev));
        FPH_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const FloodArgs& a = rp.a;
        switch (rp.ppt) {
#define FPH_LAUNCH(PPTV)                                                                     \
    case PPTV:                                                                               \
        FPH_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_kernel<PPTV>,  \
                                                                   kThreads, 0));            \
        pass_kernel<PPTV><<<sms * (occ > 0 ? occ : 1), kThreads, 0, stream>>>(               \
            a, rp.d_geom, rp.d_task_off, rp.d_counter, rp.d_done);                           \
        break;
            FPH_LAUNCH(1)
            FPH_LAUNCH(2)
            FPH_LAUNCH(4)
            FPH_LAUNCH(8)
#undef FPH_LAUNCH
        }
    }
    FPH_CUDA_TRY(cudaGetLastError());
    if (rp.profile) {
        FPH_CUDA_TRY(cudaEventRecord(ev1, stream));
        profile_push(ev0, ev1);
    }
    for (void* p : {(void*)rp.d_geom, (void*)rp.d_ntasks, (void*)rp.d_task_off,
                    (void*)rp.d_counter, (void*)rp.d_done, (void*)rp.d_perpoint, rp.tmp,
                    (void*)rp.d_cand})
        if (p) FPH_CUDA_TRY(cudaFreeAsync(p, stream));
    rp = RangePlan{};
    return FPH_OK;
}

}  // namespace

struct FloodJob {
    std::vector<RangePlan> ranges;
};

int flood_interior_prepare(const Grid* d_grid, const double* d_landmarks3, const int* d_simplices,
                           int n, int k, int m, int subset, double* d_out_sq,
                           const FloodTuning& tune, cudaStream_t stream, FloodJob** job,
                           const double* d_explicit, int explicit_rows) {
    *job = nullptr;
    if (n == 0) return FPH_OK;
    if (d_explicit && explicit_rows < 1) {
        set_error("flood_interior: explicit samples need at least one row per simplex");
        return FPH_EARG;
    }
    if (k < 0 || k > 3 || m < 1 || m > kMaxResolution) {
        set_error("flood_interior: need 0 <= k <= 3 and 1 <= m <= %d", kMaxResolution);
        return FPH_EARG;
    }
    const long long rows = d_explicit ? explicit_rows : interior_rows(k, m);
    if (rows >= (1ll << 24)) {
        set_error("grid_resolution %d gives %lld interior rows per %d-simplex (limit 2^24)", m,
                  rows, k);
        return FPH_EARG;
    }
    if (rows == 0) {
        no_interior_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_out_sq, n);
        FPH_CUDA_TRY(cudaGetLastError());
        return FPH_OK;
    }
    Template T;
    FPH_TRY(get_template(k, m, d_explicit ? explicit_rows : 0, &T));
    // simplices in chunks whose per-row scratch fits the budget (only very
    // high resolutions ever need more than one; their chunks run in turn)
    const long long chunk =
        std::max(1ll, std::min((long long)n, (long long)(kPerpointBudget / (4.0 * T.P))));
    FloodJob* jb = new FloodJob;
    for (long long off = 0; off < n; off += chunk) {
        const int cnt = (int)std::min(chunk, n - off);
        jb->ranges.emplace_back();
        const int rc = range_prepare(d_grid, d_landmarks3, d_simplices + off * 4, cnt, k, m, subset,
                                     d_out_sq + off, tune, stream,
                                     d_explicit ? d_explicit + off * (long long)T.P * 3 : nullptr,
                                     T, &jb->ranges.back());
        if (rc != FPH_OK) {
            delete jb;
            return rc;
        }
        if (off + chunk < n) {  // later chunks reuse nothing: run this one now
            const int rr = range_run(jb->ranges.back());
            if (rr != FPH_OK) {
                delete jb;
                return rr;
            }
            jb->ranges.pop_back();
        }
    }
    *job = jb;
    return FPH_OK;
}

int flood_interior_run(FloodJob* job) {
    if (!job) return FPH_OK;
    int rc = FPH_OK;
    for (RangePlan& rp : job->ranges)
        if (rc == FPH_OK) rc = range_run(rp);
    delete job;
    return rc;
}

int flood_interior(const Grid* d_grid, const double* d_landmarks3, const int* d_simplices, int n,
                   int k, int m, int subset, double* d_out_sq, const FloodTuning& tune,
                   cudaStream_t stream, const double* d_explicit, int explicit_rows) {
    FloodJob* job = nullptr;
    FPH_TRY(flood_interior_prepare(d_grid, d_landmarks3, d_simplices, n, k, m, subset, d_out_sq,
                                   tune, stream, &job, d_explicit, explicit_rows));
    return flood_interior_run(job);
}

// value(s) = max(interior(s), max_j value(facet_j(s))) -- the face-nesting
// identity that replaces the reference's per-cell face extraction
// (floodph/filtration.py:227 _extract_faces).
__global__ void complete_kernel(const double* __restrict__ interior, const int* __restrict__ facets,
                                int n, int k, const double* __restrict__ lower,
                                double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = interior[i];
    for (int j = 0; j <= k; ++j) v = fmax(v, lower[facets[(size_t)i * (k + 1) + j]]);
    out[i] = v;
}

int flood_complete(const double* d_interior, const int* d_facets, int n, int k,
                   const double* d_lower, double* d_out, cudaStream_t stream) {
    if (n == 0) return FPH_OK;
    complete_kernel<<<(n + 255) / 256, 256, 0, stream>>>(d_interior, d_facets, n, k, d_lower,
                                                         d_out);
    FPH_CUDA_TRY(cudaGetLastError());
    return FPH_OK;
}

}  // namespace fph
