/*
 * floodph_b200.h -- C ABI of the B200 flood-filtration library
 * (paper_2509_22432_b200/csrc -> libfloodph_b200.so).
 *
 * Plain pointers and sizes only.  Every entry point takes a `memory` flag:
 *   FPH_MEM_HOST    all array arguments are host pointers; the call copies
 *                   them to the GPU, runs, copies results back and returns
 *                   when they are ready (the drop-in for the CPU reference);
 *                   it runs on a stream of the calling thread, so calls from
 *                   different host threads overlap on the device;
 *   FPH_MEM_DEVICE  all data arrays (coordinates, simplices, facets, values,
 *                   indices) are device pointers on the current CUDA device;
 *                   work is ordered on `stream` (a cudaStream_t, NULL =
 *                   legacy default stream).  `counts` and the per-dimension
 *                   pointer tables (simplices[k], facets[k], out_sq[k]) are
 *                   always host arrays (their entries follow `memory`).
 * Return value: FPH_OK (0) or an FPH_E* code; fph_last_error() describes the
 * most recent failure of the calling thread.  Argument errors (FPH_EARG)
 * correspond to the reference's ValueError, FPH_EINTEGRITY to IntegrityError.
 *
 * Coordinates are float64 row-major (n x dim, dim in {2, 3}); grid_resolution
 * is any m in [1, 65535] (rows per k-simplex C(m-1, k) < 2^24); results are
 * bit-identical to the reference's float64 values.
 */
#ifndef FLOODPH_B200_H
#define FLOODPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPH_OK 0
#define FPH_EARG 1
#define FPH_ECUDA 2
#define FPH_ENOMEM 3
#define FPH_EINTEGRITY 4

#define FPH_MEM_HOST 0
#define FPH_MEM_DEVICE 1

#define FPH_ABI_VERSION 1

/* ABI version (FPH_ABI_VERSION). */
int fph_abi_version(void);

/* Message of the calling thread's last failure ("" if none). */
const char* fph_last_error(void);

/* Number of visible CUDA devices (0 when no GPU/driver). */
int fph_device_count(void);

/*
 * Farthest point sampling.
 * Replaces floodph/geometry.py:88  farthest_point_sampling(cloud, k, start):
 * out_indices[0] = start, then greedily the point maximising the distance to
 * the chosen prefix, ties to the smallest index.  Errors: k < 1, k > n or
 * start outside [0, n) -> FPH_EARG.
 */
int fph_farthest_point_sampling(const double* points, int64_t n, int32_t dim, int64_t k,
                                int64_t start, int64_t* out_indices, int32_t memory,
                                void* stream);

/*
 * Batched farthest point sampling over `batch` clouds of equal size
 * (points: batch x n x dim).  out_indices: batch x k.  Same semantics per
 * cloud as fph_farthest_point_sampling.
 */
int fph_farthest_point_sampling_batched(const double* points, int64_t batch, int64_t n,
                                        int32_t dim, int64_t k, int64_t start,
                                        int64_t* out_indices, int32_t memory, void* stream);

/*
 * Squared flood value of k-simplices over their relative-interior grid rows.
 * The kernel boundary that replaces the per-cell masked minimisation of
 * floodph/filtration.py:233 _grid_values_masked (mask: filtration.py:130
 * compute_mask; distance kernel: floodph/_kernels.py:58 min_sq_dists):
 *   out_sq[i] = max over rows c/m of simplex i with every c_j >= 1 of
 *               min over cloud points x of |x - p(c)|^2
 * (k = 0: the vertex itself; no such row, i.e. m <= k: -1).
 * simplices: n_simplices x 4 int32 landmark ids, slots > k ignored.
 * subset_mode = 1 when the landmarks are cloud points (Lemma 4.2 pruning is
 * then exact); 0 searches the whole cloud (the reference's kdtree route,
 * filtration.py:274).
 */
int fph_flood_interior(const double* points, int64_t n_points, int32_t dim,
                       const double* landmarks, int64_t n_landmarks, const int32_t* simplices,
                       int64_t n_simplices, int32_t k, int32_t grid_resolution,
                       int32_t subset_mode, double* out_sq, int32_t memory, void* stream);

/*
 * Squared flood value of k-simplices over EXPLICIT sample points: out_sq[i]
 * = max over the n_samples rows samples[i][*] (n_simplices x n_samples x
 * dim float64, inside conv(simplex i)) of min over cloud points of the
 * squared distance.  The device half of the reference's uniform-random
 * sampler (floodph/filtration.py:303 _random_sampler_values: per simplex,
 * its vertices plus Dirichlet samples, valued by exact nearest neighbours).
 */
int fph_flood_samples(const double* points, int64_t n_points, int32_t dim,
                      const double* landmarks, int64_t n_landmarks, const int32_t* simplices,
                      int64_t n_simplices, int32_t k, const double* samples, int32_t n_samples,
                      int32_t subset_mode, double* out_sq, int32_t memory, void* stream);

/*
 * Squared flood values of a whole Delaunay complex.
 * Replaces the msq_by_dim produced by floodph/filtration.py:233
 * _grid_values_masked (and :274 _grid_values_kdtree for external landmarks)
 * inside build_flood_filtration (filtration.py:348).
 *   counts[k]     number of k-simplices, k = 0..max_dim
 *   simplices[k]  counts[k] x (k+1) int32 sorted vertex ids (k >= 1; [0] unused)
 *   facets[k]     counts[k] x (k+1) int32 row of the facet dropping vertex j
 *                 in dimension k-1 (Triangulation.facet_links; [0] unused)
 *   out_sq[k]     counts[k] float64 squared values (vertices: 0 in subset mode)
 */
int fph_flood_filtration(const double* points, int64_t n_points, int32_t dim,
                         const double* landmarks, int64_t n_landmarks, int32_t max_dim,
                         const int64_t* counts, const int32_t* const* simplices,
                         const int32_t* const* facets, int32_t grid_resolution,
                         int32_t subset_mode, double* const* out_sq, int32_t memory,
                         void* stream);

/*
 * One rank's share of a sharded fph_flood_filtration: builds the grid once
 * and values the interior term of rows rank, rank + world, ... of every
 * dimension 1..max_dim; out_interior[k] receives ceil((counts[k] - rank) /
 * world) squared values in that order.  After an all-gather back into row
 * order, fph_flood_complete folds in the facets (vertices: 0 in subset
 * mode).  counts / simplices / out_interior tables are host arrays.
 */
int fph_flood_shard(const double* points, int64_t n_points, int32_t dim,
                    const double* landmarks, int64_t n_landmarks, int32_t max_dim,
                    const int64_t* counts, const int32_t* const* simplices, int32_t rank,
                    int32_t world, int32_t grid_resolution, int32_t subset_mode,
                    double* const* out_interior, int32_t memory, void* stream);

/*
 * Interior terms of an explicit subset of every dimension's simplices, with
 * one grid build: rows[k] lists n_rows[k] row indices (int64, in range) into
 * simplices[k]; out_interior[k] receives n_rows[k] squared values in that
 * order.  The general form of fph_flood_shard: a multi-GPU caller picks any
 * partition of the rows -- e.g. spatially compact shards, so each GPU's
 * working set of the cloud stays in its L2 (parallel.spatial_partition).
 * counts / simplices / rows / n_rows / out_interior are host tables whose
 * entries follow `memory`.
 */
int fph_flood_subset(const double* points, int64_t n_points, int32_t dim,
                     const double* landmarks, int64_t n_landmarks, int32_t max_dim,
                     const int64_t* counts, const int32_t* const* simplices,
                     const int64_t* const* rows, const int64_t* n_rows, int32_t grid_resolution,
                     int32_t subset_mode, double* const* out_interior, int32_t memory,
                     void* stream);

/*
 * Facet completion for sharded runs (device memory only): out[i] =
 * max(interior_sq[i], lower_sq[facets[i][j]] for j <= k).  This is the
 * face-nesting identity that replaces the reference's per-cell face
 * extraction (floodph/filtration.py:227 _extract_faces).
 */
int fph_flood_complete(const double* interior_sq, const int32_t* facets, int64_t n, int32_t k,
                       const double* lower_sq, double* out_sq, void* stream);

/*
 * Candidate masks (host memory only).  Replaces floodph/filtration.py:130
 * compute_mask -> CandidateMask (filtration.py:88): for each of n_cells
 * k-simplices (cells: n_cells x (k+1) int32 landmark ids), the ascending
 * cloud indices x with |x - c|^2 <= 2 r r, (c, r) the simplex's Ritter ball
 * (geometry.py:123), the same float64 test as the reference.
 *   out_offsets  n_cells + 1 CSR offsets (always written)
 *   out_indices  the concatenated lists, written only when capacity >= the
 *                total (call once with capacity 0 to size the buffer)
 * The reference's fallback for an empty ball (the batch slab, then the whole
 * cloud) depends on its batching and is left to the caller.
 */
int fph_candidate_mask(const double* points, int64_t n_points, int32_t dim,
                       const double* landmarks, int64_t n_landmarks, const int32_t* cells,
                       int64_t n_cells, int32_t k, int64_t* out_offsets, int32_t* out_indices,
                       int64_t capacity);

/*
 * Persistence pairs of a filtered complex (host computation, no GPU needed):
 * Z/2 column reduction with the twist / clearing optimisation.  Replaces
 * floodph/persistence.py:89 _run_reduction (pairing as :118 reduce_and_extract).
 *   counts[k], facets[k]  as in fph_flood_filtration (k = 0..max_dim)
 *   order[i]               rank of simplex i, simplices concatenated by
 *                          dimension (FilteredComplex.order)
 *   out_pairs              (birth rank, death rank) pairs, room for
 *                          sum(counts) pairs; n_pairs receives their number
 * Unpaired ranks are the essential classes.  FPH_EINTEGRITY if a facet does
 * not precede its coface.
 */
int fph_persistence_pairs(int32_t max_dim, const int64_t* counts, const int32_t* const* facets,
                          const int64_t* order, int32_t clearing, int64_t* out_pairs,
                          int64_t* n_pairs);

/*
 * Tuning knobs (<= 0 keeps the default): target points per grid cell if the
 * cloud filled its bounding box, and fp32 pairs per flood task.
 */
int fph_set_tuning(double cell_occupancy, double pairs_per_task);

/*
 * Flooding algorithm: 1 (default) bounded search -- per simplex, sampled
 * upper bounds, an exact lower bound, and exact search of only the point
 * blocks that can still hold the maximum; 0 brute force over every point of
 * the Lemma-4.2 ball.  Both are exact (identical values).
 * reps_target: candidates per representative (sampling) pass;
 * team_threshold: simplices with more candidates are searched by a whole
 * CTA instead of one warp; 0 (default) derives it per launch as
 * beta x (total candidates / resident warps) with beta = 2, a negative value
 * -b uses beta = b / 100.  reps_target <= 0 keeps the default 512.
 */
int fph_set_search(int32_t algo, int32_t reps_target, int32_t team_threshold);

/*
 * Bounded search: a simplex whose rows x candidates <= pairs is finished by
 * one exact pass (phase A unsampled) instead of the bounded search
 * (default 65536; negative restores the default).
 */
int fph_set_exact_pairs(double pairs);

/* ... and k-simplices with at most `candidates` candidates (0: off). */
int fph_set_exact_candidates(int32_t k, int64_t candidates);

/* Time every flooding-kernel launch with CUDA events (profiling aid). */
int fph_set_profiling(int32_t on);

/*
 * Work counters since the last reset: out[0] fp32 (point, candidate) pairs
 * evaluated, [1] candidates staged, [2] candidates scanned, [3] refined
 * points, [4] float64 refine distances, [5] tasks, [6] flooding-kernel ms
 * (with profiling on); block search: [7] blocks, [8] blocks pruned whole,
 * [9] points certified in round 1, [10] points still needed after round 1,
 * [11] representative passes, [12] round-2 passes, [13..15] candidates
 * scanned in round 1 / representative / round 2, [16..18] staged likewise,
 * [19..22] warp-cycles spent in the bounded search's phases A, B, C and
 * finalize.  out must hold 24 doubles.
 */
int fph_flood_stats(double* out, int32_t reset);

/*
 * Profiling aid.  n != NULL: first waits for the device and returns the
 * capture so far in out (cap int64s; out NULL: size only, *n = values
 * available) as blocks [k, count, count x 16 values], one block per flooding
 * launch; then enable (1, clearing the capture) / disable (0) capturing.
 * Per simplex: cycles in the phase kernels A, B, C, F (claim to publish);
 * blocks searched; candidate count; candidates staged; team size; global
 * timer (ns) start and end in A, B, C, F.
 */
int fph_debug_simplex_cycles(int32_t enable, int64_t* out, int64_t cap, int64_t* n);

/* Measured FP32 (FFMA2) throughput of the current device, TFLOP/s. */
double fph_fp32_peak_tflops(void);

/*
 * Tensor-core decision microbenchmarks: elements
 * per second that can leave TMEM through tcgen05.ld and be min-reduced
 * (all SMs), and (sample point, candidate) pairs per second of the FFMA2
 * tile-min loop the flooding kernel runs.  0 on failure.
 */
double fph_tmem_min_rate(void);
double fph_tilemin_rate(void);

/* Kernel launches issued by this thread since the last reset (for bench accounting). */
int64_t fph_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif

#endif /* FLOODPH_B200_H */
