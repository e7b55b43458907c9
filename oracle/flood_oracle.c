/*
 * flood_oracle.c -- CPU restatement of the reference's flood-filtration hot
 * path.  TEST INFRASTRUCTURE ONLY: the product (paper_2509_22432_b200) never
 * links or calls this file.  It is used by tests/ as the parity checker and by
 * bench.py's cpu_baseline / --impl reference leg as the CPU timing.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/<case>.npz, checked in
 * tests/test_oracle_golden.py).
 *
 * Arithmetic follows the reference exactly so results are bit-identical:
 *   - every squared distance is  s = d0*d0; s = s + d1*d1; s = s + d2*d2
 *     with d = a - b, no fused multiply-add (compile with -ffp-contract=off)
 *       reference: floodph/geometry.py:61 _coordinate_sq_sum,
 *                  floodph/_kernels.py:41 _min_sq_dists_nb
 *   - grid rows are  p = w0*v0; p = p + w1*v1; ...  with w = c / m
 *       reference: floodph/geometry.py:178 barycentric_grid_template,
 *                  floodph/geometry.py:200 barycentric_grid
 *   - Ritter ball: center = 0.5*(vi+vj) of the first longest edge in
 *     combinations order, radius = sqrt(max_i |v_i - c|^2)
 *       reference: floodph/geometry.py:123 ritter_enclosing_ball
 *   - mask: axis slab [c_a - s, c_a + s] with s = sqrt(2) r (1+1e-12), then
 *     closed ball |x - c|^2 <= 2 r r; empty -> slab -> whole cloud
 *       reference: floodph/filtration.py:130 compute_mask
 *   - per top cell: min over candidates for every grid row, then each owned
 *     face takes the max over the rows supported on it
 *       reference: floodph/filtration.py:233 _grid_values_masked,
 *                  filtration.py:227 _extract_faces
 *   - farthest point sampling with the -1 sentinel and first-index argmax
 *       reference: floodph/geometry.py:88 farthest_point_sampling
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

#define ORC_OK 0
#define ORC_EARG 1
#define ORC_ENOMEM 2

static inline double sqd(const double* a, const double* b, int dim) {
    double t = a[0] - b[0];
    double s = t * t;
    for (int k = 1; k < dim; ++k) {
        t = a[k] - b[k];
        double u = t * t;
        s = s + u;
    }
    return s;
}

/* -------------------------------------------------------- thread pool */

typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi, int tid);

typedef struct {
    range_fn fn;
    void* ctx;
    int64_t n, chunk;
    _Atomic int64_t next;
    int tid;
} par_job;

typedef struct { par_job* job; int tid; } par_arg;

static void* par_worker(void* p) {
    par_arg* a = (par_arg*)p;
    par_job* j = a->job;
    for (;;) {
        int64_t lo = atomic_fetch_add(&j->next, j->chunk);
        if (lo >= j->n) break;
        int64_t hi = lo + j->chunk < j->n ? lo + j->chunk : j->n;
        j->fn(j->ctx, lo, hi, a->tid);
    }
    return NULL;
}

static int resolve_threads(int nthreads) {
    if (nthreads > 0) return nthreads > 256 ? 256 : nthreads;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c < 1 ? 1 : (c > 256 ? 256 : (int)c);
}

/* dynamic parallel for over [0, n) in chunks; thread ids 0..nthreads-1 */
static void par_for(int64_t n, int64_t chunk, int nthreads, range_fn fn, void* ctx) {
    if (n <= 0) return;
    if (chunk < 1) chunk = 1;
    par_job job;
    job.fn = fn; job.ctx = ctx; job.n = n; job.chunk = chunk;
    atomic_init(&job.next, 0);
    int nt = nthreads;
    if ((int64_t)nt > (n + chunk - 1) / chunk) nt = (int)((n + chunk - 1) / chunk);
    if (nt <= 1) { fn(ctx, 0, n, 0); return; }
    pthread_t th[256];
    par_arg args[256];
    for (int t = 0; t < nt; ++t) {
        args[t].job = &job; args[t].tid = t;
        if (t > 0) pthread_create(&th[t], NULL, par_worker, &args[t]);
    }
    par_worker(&args[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------ FPS */

typedef struct {
    const double* pts; double* d2; const double* q; int dim;
    double best[256]; int64_t bidx[256];
} fps_ctx;

static void fps_update(void* c, int64_t lo, int64_t hi, int tid) {
    fps_ctx* x = (fps_ctx*)c;
    double lb = x->best[tid];
    int64_t li = x->bidx[tid];
    for (int64_t i = lo; i < hi; ++i) {
        double v = sqd(x->pts + i * x->dim, x->q, x->dim);
        double cur = x->d2[i];
        if (v < cur) { x->d2[i] = v; cur = v; } /* np.minimum(d2, new): NaN-free */
        if (cur > lb || (cur == lb && i < li)) { lb = cur; li = i; }
    }
    x->best[tid] = lb;
    x->bidx[tid] = li;
}

int orc_fps(const double* pts, int64_t n, int dim, int64_t k, int64_t start,
            int nthreads, int64_t* out) {
    if (k < 1 || k > n || start < 0 || start >= n || (dim != 2 && dim != 3))
        return ORC_EARG;
    fps_ctx* x = (fps_ctx*)malloc(sizeof(fps_ctx));
    double* d2 = (double*)malloc(sizeof(double) * (size_t)n);
    if (!d2 || !x) { free(d2); free(x); return ORC_ENOMEM; }
    int nt = resolve_threads(nthreads);
    int64_t chunk = (n + 4 * nt - 1) / (4 * nt);
    if (chunk < 4096) chunk = 4096;
    for (int64_t i = 0; i < n; ++i) d2[i] = INFINITY;
    x->pts = pts; x->d2 = d2; x->dim = dim;
    int64_t cur = start;
    out[0] = start;
    for (int64_t it = 1; it <= k; ++it) {
        /* fold the newest pick into the running minimum and, in the same
         * pass, find the first maximiser (np.argmax: smallest index wins) */
        x->q = pts + cur * dim;
        d2[cur] = -1.0; /* sentinel: sq_dist(cur,cur) = 0 > -1 keeps it */
        for (int t = 0; t < 256; ++t) { x->best[t] = -INFINITY; x->bidx[t] = INT64_MAX; }
        par_for(n, chunk, nt, fps_update, x);
        if (it == k) break;
        double best = -INFINITY;
        int64_t bidx = INT64_MAX;
        for (int t = 0; t < 256; ++t)
            if (x->bidx[t] != INT64_MAX &&
                (x->best[t] > best || (x->best[t] == best && x->bidx[t] < bidx))) {
                best = x->best[t]; bidx = x->bidx[t];
            }
        out[it] = bidx;
        cur = bidx;
    }
    free(d2);
    free(x);
    return ORC_OK;
}

/* ------------------------------------------------------ grid template */

static int64_t binom(int64_t a, int64_t b) {
    if (b < 0 || b > a) return 0;
    int64_t r = 1;
    for (int64_t i = 1; i <= b; ++i) r = r * (a - b + i) / i;
    return r;
}

/* integer compositions of m into k+1 parts, lexicographic (c0 ascending first) */
static void compositions(int m, int parts, int* out /* rows x parts */) {
    int c[4] = {0, 0, 0, 0};
    int64_t row = 0;
    /* iterate lexicographically: recursive via explicit loops for parts<=4 */
    if (parts == 1) { out[0] = m; return; }
    if (parts == 2) {
        for (c[0] = 0; c[0] <= m; ++c[0]) { out[row * 2] = c[0]; out[row * 2 + 1] = m - c[0]; ++row; }
        return;
    }
    if (parts == 3) {
        for (c[0] = 0; c[0] <= m; ++c[0])
            for (c[1] = 0; c[1] <= m - c[0]; ++c[1]) {
                out[row * 3] = c[0]; out[row * 3 + 1] = c[1]; out[row * 3 + 2] = m - c[0] - c[1]; ++row;
            }
        return;
    }
    for (c[0] = 0; c[0] <= m; ++c[0])
        for (c[1] = 0; c[1] <= m - c[0]; ++c[1])
            for (c[2] = 0; c[2] <= m - c[0] - c[1]; ++c[2]) {
                out[row * 4] = c[0]; out[row * 4 + 1] = c[1]; out[row * 4 + 2] = c[2];
                out[row * 4 + 3] = m - c[0] - c[1] - c[2]; ++row;
            }
}

int64_t orc_grid_size(int k, int m) { return binom(m + k, k); }

/* Embed every template row of a (k)-simplex: p = w0*v0; p = p + w_j*v_j. */
static void embed(const int* counts, int64_t rows, int k, int m, const double* verts,
                  int dim, double* out) {
    double fm = (double)m;
    for (int64_t r = 0; r < rows; ++r) {
        for (int a = 0; a < dim; ++a) {
            double w = (double)counts[r * (k + 1)] / fm;
            double p = w * verts[a];
            for (int j = 1; j <= k; ++j) {
                double wj = (double)counts[r * (k + 1) + j] / fm;
                double t = wj * verts[j * dim + a];
                p = p + t;
            }
            out[r * dim + a] = p;
        }
    }
}

/* public helper for tests: the embedded grid of one simplex */
int orc_barycentric_grid(int k, int m, const double* verts, int dim, double* out) {
    if (k < 0 || k > 3 || m < 1) return ORC_EARG;
    int64_t rows = binom(m + k, k);
    int* counts = (int*)malloc(sizeof(int) * (size_t)rows * (k + 1));
    if (!counts) return ORC_ENOMEM;
    compositions(m, k + 1, counts);
    embed(counts, rows, k, m, verts, dim, out);
    free(counts);
    return ORC_OK;
}

/* ------------------------------------------------------ Ritter ball */

static double ritter(const double* verts, int s, int dim, double* center) {
    double best = -1.0;
    int bi = 0, bj = 1;
    for (int i = 0; i < s; ++i)
        for (int j = i + 1; j < s; ++j) {
            /* float(np.sum((vi - vj) ** 2)): sequential sum of squares */
            double acc = 0.0;
            for (int a = 0; a < dim; ++a) {
                double t = verts[i * dim + a] - verts[j * dim + a];
                double u = t * t;
                acc = acc + u;
            }
            if (acc > best) { best = acc; bi = i; bj = j; }
        }
    for (int a = 0; a < dim; ++a) center[a] = 0.5 * (verts[bi * dim + a] + verts[bj * dim + a]);
    double mx = -1.0;
    for (int i = 0; i < s; ++i) {
        double acc = 0.0;
        for (int a = 0; a < dim; ++a) {
            double t = verts[i * dim + a] - center[a];
            double u = t * t;
            acc = acc + u;
        }
        if (acc > mx) mx = acc;
    }
    return sqrt(mx);
}

int orc_ritter(const double* verts, int s, int dim, double* center, double* radius) {
    if (s < 2) return ORC_EARG;
    *radius = ritter(verts, s, dim, center);
    return ORC_OK;
}

/* ------------------------------------------------ masked cell values */

typedef struct { double key; int64_t idx; } keyed;

static int cmp_keyed(const void* a, const void* b) {
    const keyed* x = (const keyed*)a;
    const keyed* y = (const keyed*)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx); /* stable */
}

static int64_t lower_bound(const double* v, int64_t n, double x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (v[mid] < x) lo = mid + 1; else hi = mid; }
    return lo;
}
static int64_t upper_bound(const double* v, int64_t n, double x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (v[mid] <= x) lo = mid + 1; else hi = mid; }
    return lo;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/*
 * Values of every face owned by each top cell.
 *
 *   X[n*dim]                  the cloud
 *   tri_pts[*dim]             landmark coordinates (triangulation points)
 *   cells[n_cells*(kc+1)]     top cells (kc = their dimension), vertex ids
 *   face_ptr[n_cells+1]       CSR offsets into face_mask/face_out
 *   face_mask[]               bitmask of cell vertex positions spanning the face
 *   face_out[]                output slot (index into out_msq) of that face
 *   subset_mode               1: masked (Lemma 4.2) candidates; 0: whole cloud
 *   out_msq[]                 squared flood values, written per owned face
 */
typedef struct {
    const double* X; int64_t n; int dim;
    const double* tri_pts; const int64_t* cells; int kc, s; int64_t rows;
    const int* counts; const int32_t* support;
    const int64_t* face_ptr; const int32_t* face_mask; const int64_t* face_out;
    int subset_mode; int axis; int fm; const keyed* ks; const double* sorted;
    double* out_msq;
    double* grid[256]; double* msq[256]; int64_t* cand[256];
} cells_ctx;

static void cells_run(void* c, int64_t lo, int64_t hi, int tid) {
    cells_ctx* x = (cells_ctx*)c;
    const int s = x->s, dim = x->dim;
    const int64_t n = x->n, rows = x->rows;
    double* grid = x->grid[tid];
    double* msq = x->msq[tid];
    int64_t* cand = x->cand[tid];
    double verts[12];
    for (int64_t cell = lo; cell < hi; ++cell) {
        for (int j = 0; j < s; ++j)
            for (int a = 0; a < dim; ++a)
                verts[j * dim + a] = x->tri_pts[x->cells[cell * s + j] * dim + a];
        embed(x->counts, rows, x->kc, x->fm, verts, dim, grid);
        int64_t nc = 0;
        if (x->subset_mode) {
            double center[3];
            double r = ritter(verts, s, dim, center);
            double span = sqrt(2.0) * r * (1.0 + 1e-12);
            int64_t a0 = lower_bound(x->sorted, n, center[x->axis] - span);
            int64_t a1 = upper_bound(x->sorted, n, center[x->axis] + span);
            double thr = 2.0 * r * r;
            for (int64_t q = a0; q < a1; ++q) {
                int64_t i = x->ks[q].idx;
                if (sqd(x->X + i * dim, center, dim) <= thr) cand[nc++] = i;
            }
            if (nc == 0)
                for (int64_t q = a0; q < a1; ++q) cand[nc++] = x->ks[q].idx;
            qsort(cand, (size_t)nc, sizeof(int64_t), cmp_i64);
        }
        if (nc == 0) { for (int64_t i = 0; i < n; ++i) cand[i] = i; nc = n; }
        for (int64_t r = 0; r < rows; ++r) {
            const double* p = grid + r * dim;
            double best = INFINITY;
            for (int64_t q = 0; q < nc; ++q) {
                double v = sqd(x->X + cand[q] * dim, p, dim);
                if (v < best) best = v;
            }
            msq[r] = best;
        }
        for (int64_t f = x->face_ptr[cell]; f < x->face_ptr[cell + 1]; ++f) {
            int32_t fm = x->face_mask[f];
            double mx = -INFINITY;
            for (int64_t r = 0; r < rows; ++r)
                if ((x->support[r] & ~fm) == 0 && msq[r] > mx) mx = msq[r];
            x->out_msq[x->face_out[f]] = mx;
        }
    }
}

int orc_flood_cells(const double* X, int64_t n, int dim, const double* tri_pts,
                    const int64_t* cells, int64_t n_cells, int kc, int m,
                    const int64_t* face_ptr, const int32_t* face_mask,
                    const int64_t* face_out, int subset_mode, int nthreads,
                    double* out_msq) {
    if (kc < 1 || kc > 3 || m < 1 || (dim != 2 && dim != 3) || n < 1) return ORC_EARG;
    const int s = kc + 1;
    const int64_t rows = binom(m + kc, kc);
    int nt = resolve_threads(nthreads);
    cells_ctx* x = (cells_ctx*)calloc(1, sizeof(cells_ctx));
    int* counts = (int*)malloc(sizeof(int) * (size_t)rows * s);
    int32_t* support = (int32_t*)malloc(sizeof(int32_t) * (size_t)rows);
    keyed* ks = (keyed*)malloc(sizeof(keyed) * (size_t)n);
    double* sorted = (double*)malloc(sizeof(double) * (size_t)n);
    int err = (!x || !counts || !support || !ks || !sorted) ? ORC_ENOMEM : ORC_OK;
    if (err == ORC_OK) {
        compositions(m, s, counts);
        for (int64_t r = 0; r < rows; ++r) {
            int32_t b = 0;
            for (int j = 0; j < s; ++j) if (counts[r * s + j] != 0) b |= 1 << j;
            support[r] = b;
        }
        /* axis-sorted view along the widest axis (reference spatial.py:34,38) */
        int axis = 0;
        double ext_best = -1.0;
        for (int a = 0; a < dim; ++a) {
            double lo = X[a], hi = X[a];
            for (int64_t i = 1; i < n; ++i) { double v = X[i * dim + a]; if (v < lo) lo = v; if (v > hi) hi = v; }
            if (hi - lo > ext_best) { ext_best = hi - lo; axis = a; }
        }
        for (int64_t i = 0; i < n; ++i) { ks[i].key = X[i * dim + axis]; ks[i].idx = i; }
        qsort(ks, (size_t)n, sizeof(keyed), cmp_keyed);
        for (int64_t i = 0; i < n; ++i) sorted[i] = ks[i].key;
        x->X = X; x->n = n; x->dim = dim; x->tri_pts = tri_pts; x->cells = cells;
        x->kc = kc; x->s = s; x->rows = rows; x->counts = counts; x->support = support;
        x->face_ptr = face_ptr; x->face_mask = face_mask; x->face_out = face_out;
        x->subset_mode = subset_mode; x->axis = axis; x->ks = ks; x->sorted = sorted;
        x->out_msq = out_msq;
        x->fm = m;
        for (int t = 0; t < nt && err == ORC_OK; ++t) {
            x->grid[t] = (double*)malloc(sizeof(double) * (size_t)rows * dim);
            x->msq[t] = (double*)malloc(sizeof(double) * (size_t)rows);
            x->cand[t] = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
            if (!x->grid[t] || !x->msq[t] || !x->cand[t]) err = ORC_ENOMEM;
        }
        if (err == ORC_OK) par_for(n_cells, 1, nt, cells_run, x);
        for (int t = 0; t < nt; ++t) { free(x->grid[t]); free(x->msq[t]); free(x->cand[t]); }
    }
    free(counts); free(support); free(ks); free(sorted); free(x);
    return err;
}

/* ------------------------------------------- definition-level value */

/*
 * Squared flood value of single simplices straight from the definition:
 * max over the simplex's own grid rows of min over the WHOLE cloud.  Used by
 * tests as the unmasked cross-check (reference test_filtration.py
 * test_masking_invariance_against_unmasked) and for the external-landmark
 * path (reference filtration.py:274, which queries exact nearest neighbours).
 */
typedef struct {
    const double* X; int64_t n; int dim; const double* tri_pts;
    const int64_t* simp; int k, m; int64_t rows; const int* counts;
    double* out; double* grid[256];
} unmasked_ctx;

static void unmasked_run(void* c, int64_t lo, int64_t hi, int tid) {
    unmasked_ctx* x = (unmasked_ctx*)c;
    const int s = x->k + 1, dim = x->dim;
    double verts[12];
    double* grid = x->grid[tid];
    for (int64_t c2 = lo; c2 < hi; ++c2) {
        for (int j = 0; j < s; ++j)
            for (int a = 0; a < dim; ++a)
                verts[j * dim + a] = x->tri_pts[x->simp[c2 * s + j] * dim + a];
        embed(x->counts, x->rows, x->k, x->m, verts, dim, grid);
        double mx = -INFINITY;
        for (int64_t r = 0; r < x->rows; ++r) {
            double best = INFINITY;
            for (int64_t i = 0; i < x->n; ++i) {
                double v = sqd(x->X + i * dim, grid + r * dim, dim);
                if (v < best) best = v;
            }
            if (best > mx) mx = best;
        }
        x->out[c2] = mx;
    }
}

int orc_flood_unmasked(const double* X, int64_t n, int dim, const double* tri_pts,
                       const int64_t* simplices, int64_t n_simp, int k, int m,
                       int nthreads, double* out_msq) {
    if (k < 0 || k > 3 || m < 1 || (dim != 2 && dim != 3)) return ORC_EARG;
    const int s = k + 1;
    const int64_t rows = binom(m + k, k);
    int nt = resolve_threads(nthreads);
    unmasked_ctx* x = (unmasked_ctx*)calloc(1, sizeof(unmasked_ctx));
    int* counts = (int*)malloc(sizeof(int) * (size_t)rows * s);
    int err = (!x || !counts) ? ORC_ENOMEM : ORC_OK;
    if (err == ORC_OK) {
        compositions(m, s, counts);
        x->X = X; x->n = n; x->dim = dim; x->tri_pts = tri_pts; x->simp = simplices;
        x->k = k; x->m = m; x->rows = rows; x->counts = counts; x->out = out_msq;
        for (int t = 0; t < nt && err == ORC_OK; ++t) {
            x->grid[t] = (double*)malloc(sizeof(double) * (size_t)rows * dim);
            if (!x->grid[t]) err = ORC_ENOMEM;
        }
        if (err == ORC_OK) par_for(n_simp, 1, nt, unmasked_run, x);
        for (int t = 0; t < nt; ++t) free(x->grid[t]);
    }
    free(counts); free(x);
    return err;
}
