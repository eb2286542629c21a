/*
 * filterreg_b200.h -- C ABI of the B200 FilterReg engine (libfilterreg_b200.so).
 *
 * The reference (`twistreg`, /root/reference/pkg/src/twistreg) is pure Python;
 * its "operator API" for the hot path is the Python lattice / moment / solver
 * surface.  Each entry point below replaces one of those operators and cites
 * the reference symbol (file:line, relative to pkg/src/twistreg/).  The Python
 * package `paper_1811_10136_b200` binds these with ctypes exactly the way a
 * maintainer would bind them from twistreg.
 *
 * Conventions
 *  - Every pointer argument named d_* is DEVICE memory on the current CUDA
 *    device, owned by the caller, contiguous, borrowed for the call.
 *  - Every call is ordered on `stream` (a cudaStream_t passed as void*; NULL =
 *    legacy default stream) and spawns no host threads.  Calls that must size
 *    internal buffers (splat, blur) synchronise `stream` internally.
 *  - Return value: FR_OK or an FR_E* status; fr_last_error() returns the
 *    thread-local message of the last failure.  Status -> Python exception:
 *      FR_EINVAL   -> ValueError          (permutohedral.py:57-60, 148-149, 222-225)
 *      FR_ESTATE   -> RuntimeError        (permutohedral.py:301-302, 331-332)
 *      FR_EDEGEN   -> DegenerateCorrespondenceError (estep.py:256-257)
 *      FR_ESOLVER  -> SolverError         (mstep.py:368-369)
 *      FR_ECAPACITY / FR_ECUDA -> RuntimeError
 *  - An fr_lattice is single-writer during splat/blur and immutable after
 *    blur; slicing from several streams concurrently is then safe.
 */
#ifndef FILTERREG_B200_H
#define FILTERREG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    FR_OK = 0,
    FR_EINVAL = 1,
    FR_ESTATE = 2,
    FR_EDEGEN = 3,
    FR_ESOLVER = 4,
    FR_ECAPACITY = 5,
    FR_ECUDA = 6
};

/* value_mode bits for fr_lattice_splat_points: which observation-derived
 * columns are splatted, in the reference's order [1, y, (|y|^2), (n)]
 * (estep.py:153-165). */
enum {
    FR_VALUES_M2 = 1,       /* append |y|^2 (update_sigma) */
    FR_VALUES_NORMALS = 2,  /* append the observation normal (point_to_plane) */
    /* site sums in np.add.at's flat (point, vertex) order, bit-identical to the
     * reference's splat (permutohedral.py:241-242).  Without it the point
     * splats sum each site's entries in a fixed tree order (deterministic,
     * float64 round-off from the flat order, a serial chain of cnt / 256
     * adds instead of cnt). */
    FR_SPLAT_FLAT_ORDER = 256,
    /* the points are spatially ordered (e.g. Morton-sorted): consecutive
     * points' vertex contributions are folded per site inside each warp
     * before the sort (tree order, deterministic; far fewer sort items).  A
     * cloud without such locality falls back to the per-entry path. */
    FR_SPLAT_SPATIAL = 512
};

/* residual modes (mstep.py:33) */
enum { FR_POINT_TO_POINT = 0, FR_POINT_TO_PLANE = 1 };

typedef struct fr_lattice fr_lattice;

int fr_abi_version(void);
const char *fr_last_error(void);

/* ---- permutohedral lattice (permutohedral.py:140-345) ------------------- */

/* PermutohedralLattice(dim, sigma) (permutohedral.py:147-167); sigma has dim
 * host doubles, dim in 1..12 (d <= 3: hashed 63-bit keys; 4..12: sorted
 * 128-bit keys).  Destroy is stream-ordered: the buffers return to the device
 * pool behind the work enqueued on the stream of the last build call
 * (splat / blur); callers that slice from other streams synchronise those
 * streams before destroying. */
int fr_lattice_create(int dim, const double *sigma, fr_lattice **out);
int fr_lattice_destroy(fr_lattice *lat);

/* Re-bind the stream the lattice's stream-ordered frees (destroy, rebuild) go
 * behind -- for a lattice built on a side stream and then used on another
 * (the build must be complete, e.g. that stream synchronised).  Engine-
 * internal lifetime control; no reference counterpart. */
int fr_lattice_set_stream(fr_lattice *lat, void *stream);

/* PermutohedralLattice.splat(features, values) (permutohedral.py:219-251):
 * d_features n x dim row-major float64, d_values n x nv row-major float64.
 * Deterministic: per-site sums run in flat (point, vertex) order, bit-identical
 * to the reference's np.add.at. */
int fr_lattice_splat(fr_lattice *lat, const double *d_features, const double *d_values,
                     int64_t n, int nv, void *stream);

/* Same, with the value columns generated on the fly from float32 SoA point
 * planes (d_pos: 3 planes of n floats; d_normals likewise or NULL):
 * [1, y, (|y|^2 if FR_VALUES_M2), (n if FR_VALUES_NORMALS)] (estep.py:153-165). */
int fr_lattice_splat_points(fr_lattice *lat, const float *d_pos, const float *d_normals,
                            int64_t n, int value_mode, void *stream);
/* fr_upload_points + fr_lattice_splat_points (positions only, value columns
 * [1, y] or [1, y, |y|^2]) in one call: each staged chunk's splat entries run
 * as soon as its copy lands, overlapping the rest of the upload.  d_soa
 * receives the (3, n) float32 planes as from fr_upload_points.  `uploaded`
 * (nullable) is called with `ctx` on the calling thread once the host-side
 * staging is done (the staged-upload slots are free for another upload)
 * while the rest of the splat is still being enqueued. */
int fr_lattice_splat_upload(fr_lattice *lat, const double *host_xyz, int64_t n, int value_mode,
                            float *d_soa, void *stream, void (*uploaded)(void *), void *ctx);

/* fr_upload_rows64 + fr_lattice_splat_points on the float64 planes (positions
 * in the caller's order, value columns [1, y] or [1, y, |y|^2]) in one call.
 * Page-locked rows of >= 256k points go out as up to 8 back-to-back copies on
 * an internal copy stream (after the work already on `stream`); each range's
 * transpose into d_soa and its splat entries run on a side stream as soon as
 * the range lands, under the remaining copies.  Once every copy is enqueued,
 * `follow_stream` (nullable) is made to wait for them (the caller's next
 * transfer does not share the link with them) and `uploaded` (nullable) is
 * called with `ctx`.  Sums, keys and sites are those of fr_upload_rows64 +
 * fr_lattice_splat_points; on return `stream` is ordered after all of it. */
int fr_lattice_splat_rows64(fr_lattice *lat, const double *host_xyz, int64_t n, int value_mode,
                            double *d_rows, double *d_soa, void *stream, void *follow_stream,
                            void (*uploaded)(void *), void *ctx);

/* (n, 3) float64 host rows (pageable) -> (3, n) float32 device planes, the
 * boundary conversion of PointCloud.positions / normals (geometry.py:109-139,
 * "convert once to fp32 SoA device tensors").  Rounds to
 * nearest like numpy.astype(float32).  Host helper: worker threads convert
 * sub-chunks into pinned staging slots and enqueue the copies on `stream`; the
 * host rows may be reused once the call returns. */
int fr_upload_points(const double *host_xyz, int64_t n, float *d_soa, void *stream);

/* PermutohedralLattice.blur() (permutohedral.py:291-327), incl. frontier growth
 * with the reference's site cap and the final drop of all-zero rows. */
int fr_lattice_blur(fr_lattice *lat, void *stream);

/* num_sites / value width / blurred flag (permutohedral.py:343-345). */
int fr_lattice_info(const fr_lattice *lat, int64_t *num_sites, int *nv, int *blurred);

/* Cells of the dense float32 slice grid the EM pass queries instead of the
 * hash table (d = 3, 4 value columns, site box within FR_DENSE_MAX_CELLS,
 * default 16M cells); 0 when the lattice has none.  Engine-internal
 * acceleration structure -- no reference counterpart. */
int fr_lattice_dense_cells(const fr_lattice *lat, int64_t *cells);

/* Site table export (PermutohedralLattice.keys/.values): d_keys num_sites x
 * (dim+1) int32, d_values num_sites x nv float64.  Row order is unspecified;
 * callers sort lexicographically to get the reference order. */
int fr_lattice_export(const fr_lattice *lat, int32_t *d_keys, double *d_values, void *stream);

/* PermutohedralLattice.slice(query) (permutohedral.py:329-341): d_query m x dim
 * float64 row-major -> d_out m x nv float64. */
int fr_lattice_slice(const fr_lattice *lat, const double *d_query, int64_t m, double *d_out,
                     void *stream);

/* PermutohedralLattice._simplex (permutohedral.py:181-215), bit-exact:
 * d_keys n x (dim+1) x (dim+1) int32, d_bary n x (dim+1) float64. */
int fr_simplex(int dim, const double *sigma, const double *d_features, int64_t n,
               int32_t *d_keys, double *d_bary, void *stream);

/* gaussian_transform_bruteforce (permutohedral.py:64-86): exact sums,
 * d_q m x dim, d_f n x dim, d_v n x nv, d_out m x nv (all float64). */
int fr_gauss_bruteforce(const double *d_q, int64_t m, const double *d_f, int64_t n, int dim,
                        const double *d_v, int nv, const double *sigma, double *d_out,
                        void *stream);

/* Reorder a float32 SoA cloud (d_pos: `planes` planes of n, the first three
 * x, y, z) in place along a 24-bit Morton curve of its bounding box, so that
 * neighbouring threads of the EM pass query neighbouring simplices.  The
 * permutation (new -> old index) is written to d_perm when not NULL.  Used
 * once per registration on the model points: the EM sums are order-
 * independent up to float64 round-off.  Stream-ordered on `stream` (returns
 * without waiting for the device). */
int fr_sort_points_morton(float *d_pos, int64_t n, int planes, int32_t *d_perm, void *stream);

/* ---- E step (estep.py:186-217) ------------------------------------------ */

/* MomentEngine.moments epilogue fused into the slice: d_x m x 3 float64
 * positions.  m2_col / normal_col are value-column indices or -1.  Any output
 * pointer may be NULL except d_m0, d_m1, d_weight, d_target. */
int fr_moments(const fr_lattice *lat, const double *d_x, int64_t m, double c_prime,
               int m2_col, int normal_col, double *d_m0, double *d_m1, double *d_weight,
               double *d_target, double *d_m2, double *d_normal, uint8_t *d_normal_valid,
               void *stream);


/* MomentEngine.moments epilogue alone (estep.py:195-217) over raw kernel sums
 * d_raw (m x nv float64, from fr_lattice_slice or fr_gauss_bruteforce) at model
 * positions d_x (m x 3); outputs as fr_moments. */
int fr_moments_epilogue(const double *d_raw, int64_t m, int nv, const double *d_x,
                        double c_prime, int m2_col, int normal_col, double *d_m0,
                        double *d_m1, double *d_weight, double *d_target, double *d_m2,
                        double *d_normal, uint8_t *d_normal_valid, void *stream);

/* assemble_rigid + objective (mstep.py:102-138, 179-210) over an explicit
 * ResidualSpec: d_x, d_target, d_normal m x 3 float64, d_weight m, d_valid m
 * (uint8; point_to_plane only).  d_sums receives 28 doubles:
 * [upper-triangular H (21, row-major i <= j) | g (6) | sum of squared rows]. */
int fr_assemble_rigid(const double *d_x, const double *d_weight, const double *d_target,
                      int64_t m, const double *sigma_inv, int mode, const double *d_normal,
                      const uint8_t *d_valid, double *d_sums, double *d_scratch, void *stream);

/* ---- fused rigid EM pass (pipeline.py:141-166 + mstep.py:179-210) ------- */

/* Per-iteration pose/kernel constants, all host-side float64. */
typedef struct fr_rigid_pass_params {
    double R[9];        /* current rotation, row-major */
    double c_ref[3];    /* centroid of the reference cloud (xh = x_ref - c_ref) */
    double c_world[3];  /* R c_ref + t: x = R xh + c_world */
    double sigma[3];    /* kernel widths of the lattice */
    double c_prime;     /* outlier constant (estep.py:99-112) */
    int mode;           /* FR_POINT_TO_POINT / FR_POINT_TO_PLANE */
    int m2_col;         /* value column of |y|^2 or -1 */
    int normal_col;     /* value column of the normal sum or -1 */
    int flags;          /* FR_PASS_FAST: float32 ranks / barycentrics / table rows;
                           FR_PASS_F32: + float32 coordinates / moments (pt2pt) */
} fr_rigid_pass_params;

enum { FR_PASS_FAST = 1, FR_PASS_F32 = 2 };

/* Number of float64 partial sums the pass produces for a mode. */
int fr_rigid_pass_width(int mode, int with_sigma);

/* One E step + M-step assembly over all model points at pose (R, t):
 * slice at x = R x_ref + t, moments epilogue, residual rows and the
 * normal-equation sums, reduced deterministically into d_sums
 * (fr_rigid_pass_width doubles; layout in paper_1811_10136_b200/_rigid.py).
 * d_ref: 3 float32 planes of m.  d_wtn (point_to_plane only, else NULL):
 * 7 float32 planes of m receiving weight, target, normal for the candidate
 * objective pass.  d_scratch: >= fr_rigid_scratch_doubles(mode,...) doubles. */
int fr_rigid_scratch_doubles(int mode, int with_sigma, int64_t m);
int fr_rigid_pass(const fr_lattice *lat, const float *d_ref, int64_t m,
                  const fr_rigid_pass_params *p, double *d_sums, float *d_wtn,
                  double *d_scratch, void *stream);

/* Objective of k candidate poses (mstep.py:132-138 at mstep.py:443-449) under
 * the weights/targets/normals stored by the last point_to_plane pass.
 * cand_R: k x 9, cand_c: k x 3 (R_k c_ref + t_k) host doubles; d_out: k
 * float64 values 0.5 * sum r^2 (d_out must hold 16 doubles).  k <= 16. */
int fr_rigid_objective(const float *d_ref, const float *d_wtn, int64_t m,
                       const double *c_ref, int k, const double *cand_R,
                       const double *cand_c, double *d_out, double *d_scratch,
                       void *stream);

/* ---- articulated trees (mstep.py:179-202, 213-229; kinematics.py:317-336) --
 * Model points sorted by body; chunk i = points [chunk_beg[i], chunk_beg[i+1])
 * of body chunk_body[i]; body b owns chunks [body_chunks[b], body_chunks[b+1]).
 * One pass gives per-body statistics (fr_rigid_pass_width(mode, 0) doubles
 * per body, same layout as the rigid pass, each about the body's own centre
 * c_world = R_b c_ref_b + t_b); the host projects H_b, g_b through the
 * spatial velocity Jacobians.  d_params: >= fr_body_params_doubles(n) doubles
 * (n = n_bodies for the pass, n_bodies * k for the objective). */
typedef struct fr_body_pose {
    double R[9];
    double c_ref[3];
    double c_world[3];
} fr_body_pose;

int fr_body_params_doubles(int n);
int fr_body_pass(const fr_lattice *lat, const float *d_ref, int64_t m, const fr_body_pose *poses,
                 int n_bodies, const int32_t *d_chunk_body, const int64_t *d_chunk_beg,
                 int n_chunks, const int32_t *d_body_chunks, int mode, double c_prime, int flags,
                 double *d_params, double *d_sums, float *d_wtn, double *d_scratch,
                 void *stream);
/* point_to_plane halving candidates: cand[c * n_bodies + b]; d_out 16 doubles */
int fr_body_objective(const float *d_ref, const float *d_wtn, int64_t m,
                      const fr_body_pose *cand, int n_bodies, int k,
                      const int32_t *d_chunk_body, const int64_t *d_chunk_beg, int n_chunks,
                      double *d_params, double *d_out, double *d_scratch, void *stream);

/* ---- node graphs (mstep.py:232-314, kinematics.py:254-346, geometry.py:342-368)
 * d_sidx / d_swt: m x K skinning (int32 node index, -1 padding / float64
 * weight); d_node_dq: n_nodes x 8 dual quaternions [real | dual].
 * fr_graph_pass: DQB forward map, slice + moments (respec = 0) or the stored
 * spec (respec = 1), per-point E^T E / E^T r into d_ete (m x 28), and
 * d_sums = [data objective, inlier mass, sigma numerator, sigma mass].
 * fr_graph_blocks: node diagonal blocks (n_nodes x 27: upper-21 H | g) and
 * co-skinned pair blocks (n_pairs x 21, symmetric) from the (point, slot)
 * lists d_dptr/d_dent (code p*K+slot, grouped by node) and d_pptr/d_pent
 * (pairs of int32: point, slot_a | slot_c << 8), in list order.
 * fr_graph_objective: data objectives of k <= 16 candidate node states
 * (d_cand_dq: k x n_nodes x 8) under the stored spec; d_out 16 doubles.
 * d_flag is set when a blend degenerates (DegenerateBlendError). */
int fr_graph_pass(const fr_lattice *lat, const float *d_ref, int64_t m, const int32_t *d_sidx,
                  const double *d_swt, int K, const double *d_node_dq, int mode,
                  const double *sigma_inv, double c_prime, int respec, double *d_rec,
                  double *d_ete, double *d_sums, double *d_scratch, int32_t *d_flag,
                  void *stream);
int fr_graph_blocks(const double *d_ete, const double *d_swt, int K, const int32_t *d_dptr,
                    const int32_t *d_dent, int n_nodes, const int32_t *d_pptr,
                    const int32_t *d_pent, int n_pairs, double *d_diag, double *d_off,
                    void *stream);
/* per-point [E^T E upper 21 | E^T r 6 | 0] (m x 28) of an explicit ResidualSpec
 * at explicit positions (d_x, d_target, d_normal m x 3, d_weight m, d_valid m;
 * the assemble_* API of mstep.py:179-314); feed fr_graph_blocks. */
int fr_point_rows(const double *d_x, const double *d_weight, const double *d_target,
                  const double *d_normal, const uint8_t *d_valid, int64_t m, int mode,
                  const double *sigma_inv, double *d_ete, void *stream);
int fr_graph_objective(const float *d_ref, int64_t m, const int32_t *d_sidx,
                       const double *d_swt, int K, const double *d_cand_dq, int n_nodes, int k,
                       const double *d_rec, int mode, const double *sigma_inv, double *d_out,
                       double *d_scratch, int32_t *d_flag, void *stream);

/* ---- device-resident rigid EM loop (pipeline.py:141-181, point_to_point) --
 * The whole EM iteration stays on the GPU: fused pass, fixed-order reduction,
 * and a one-thread float64 solver kernel that assembles the normal equations
 * from the pass statistics, solves with the reference's damping escalation,
 * halves steps with closed-form candidate objectives, applies the twist
 * update, records objective / twist norm / inlier mass and sets the
 * termination flag.  Iterations replay a captured CUDA graph; iterations
 * enqueued after termination are no-ops.  For a sharded run, call
 * fr_rigid_em_pass, all-reduce the fr_rigid_em_sums buffer, then
 * fr_rigid_em_solve, in the same stream order on every rank. */
typedef struct fr_rigid_em fr_rigid_em;

typedef struct fr_rigid_em_config {
    double R0[9];            /* initial pose */
    double t0[3];
    double c_ref[3];         /* centre of the whole reference cloud */
    double sigma_inv[3];     /* residual scaling 1/sigma (mstep.py:98) */
    double c_prime;          /* outlier constant */
    double diameter;         /* bbox diagonal of the whole reference cloud */
    double twist_tolerance;
    double damping;          /* < 0: 1e-6 trace(A) / n (mstep.py:358) */
    double step_tolerance;
    double degenerate_mass;  /* 1e-9 * total model points (pipeline.py:150) */
    int max_em_iters;
    int max_gn_iters;
    int max_halvings;
    int fast;                /* FR_PASS_FAST query path */
} fr_rigid_em_config;

/* termination codes of fr_rigid_em_status / fr_rigid_em_result */
enum { FR_TERM_MAX_ITERS = 0, FR_TERM_CONVERGED = 1, FR_TERM_DEGENERATE = 2,
       FR_TERM_SOLVER = 3 };

int fr_rigid_em_create(const fr_lattice *lat, const float *d_ref, int64_t m,
                       const fr_rigid_em_config *cfg, fr_rigid_em **out);
/* as fr_rigid_em_create, with the setup (allocations, the centred tiled copy
 * of d_ref for clouds above FR_PERSIST_MAX points, the first pass constants)
 * ordered on `stream` -- the stream that produced d_ref */
int fr_rigid_em_create_on(const fr_lattice *lat, const float *d_ref, int64_t m,
                          const fr_rigid_em_config *cfg, void *stream, fr_rigid_em **out);
int fr_rigid_em_destroy(fr_rigid_em *em);
/* kernels one fr_rigid_em_enqueue'd iteration launches (1: the tiled pass with
 * its fused reduction and solve) -- for launch accounting */
int fr_rigid_em_kernels_per_iter(const fr_rigid_em *em);
int fr_rigid_em_sums(fr_rigid_em *em, double **d_sums, int *width);
int fr_rigid_em_pass(fr_rigid_em *em, void *stream);
/* the tiled pass kernel alone, reusing the pass constants the last
 * fr_rigid_em_pass copied into the constant bank (kernel timing: the pose
 * must not have changed since) */
int fr_rigid_em_pass_kernel(fr_rigid_em *em, void *stream);
int fr_rigid_em_solve(fr_rigid_em *em, void *stream);
int fr_rigid_em_enqueue(fr_rigid_em *em, int n_iters, void *stream);
int fr_rigid_em_run(fr_rigid_em *em, void *stream);

/* 1 when fr_rigid_em_run takes the persistent path: the dense-grid float32
 * point pass and at most FR_PERSIST_MAX model points (default 32768).  There
 * one CTA runs the whole EM loop (pass, fixed-order reduction, float64 solve)
 * with no launches or host polls between iterations. */
int fr_rigid_em_persistent(const fr_rigid_em *em);

/* Independent registrations (replicas, no collectives) in ONE launch: CTA i
 * runs ems[i]'s EM loop to termination (the batched multi-problem driver,
 * bench.py:132-159 of the reference runs trials one after another).  Every
 * em must run the dense-grid float32 pass (FR_EINVAL otherwise); a problem's
 * result equals fr_rigid_em_run's when fr_rigid_em_persistent(em) is 1.
 * Synchronises `stream`. */
int fr_rigid_em_run_batch(fr_rigid_em **ems, int n, void *stream);
int fr_rigid_em_status(fr_rigid_em *em, int *done, int *iterations, int *termination,
                       void *stream);
/* pose, per-iteration traces (host arrays of >= max_em_iters doubles or NULL),
 * iteration count and termination; FR_ESOLVER when the solve failed. */
int fr_rigid_em_result(fr_rigid_em *em, double *R, double *t, double *objectives,
                       double *twist_norms, double *inlier_masses, int *iterations,
                       int *termination, void *stream);

/* ---- float64 device-resident rigid EM loop (pipeline.py:125-181 with the
 * reference's float64 arithmetic; point_to_point, fixed kernel width) ------
 * Model points are float64 SoA planes (d_ref: 3 planes of m, the caller's
 * values, Morton-ordered by fr_sort_points_morton64).  Every query-side
 * operation (forward map kinematics.py:317-320, elevation and simplex
 * permutohedral.py:171-215, slice permutohedral.py:329-341 over the
 * lattice's dense float64 grid, moments epilogue estep.py:195-205, the
 * point-to-point statistics of mstep.py:102-210) runs in float64; the solve
 * is the same float64 device solve as fr_rigid_em.  fr_em64_run runs up to
 * n_iters iterations (<= 0: max_em_iters) in ONE cooperative grid-resident
 * launch: pass, fixed-order reduction by the last CTA to arrive, solve, and a
 * release of the next pose to the spinning CTAs, per iteration.  Sharded
 * runs call fr_em64_pass, all-reduce fr_em64_sums, then fr_em64_solve. */
typedef struct fr_em64 fr_em64;

int fr_em64_create(const fr_lattice *lat, const double *d_ref, int64_t m,
                   const fr_rigid_em_config *cfg, void *stream, fr_em64 **out);
int fr_em64_destroy(fr_em64 *em);
int fr_em64_run(fr_em64 *em, int n_iters, void *stream);
/* one pass + fixed-order reduction at the current pose into the sums buffer
 * (no solve): kernel timing and the sharded loop */
/* independent registrations (replicas, no collectives) in ONE cooperative
 * launch, problem i on its own CTAs (the batched multi-problem driver; the
 * reference runs bench trials one after another, bench.py:132-159).
 * Synchronises `stream`. */
int fr_em64_run_batch(fr_em64 **ems, int n, void *stream);
int fr_em64_pass(fr_em64 *em, void *stream);
int fr_em64_solve(fr_em64 *em, void *stream);
/* Sharded loop, fused: one cooperative launch that first solves the previous
 * pass's sums (all-reduced in place in fr_em64_sums' buffer between the
 * launches; every CTA solves them, as in the unsharded loop), then runs this
 * iteration's pass + reduction.  Per iteration: this launch + one all-reduce;
 * fr_em64_solve after the last launch takes the final pending solve. */
int fr_em64_pass_solve(fr_em64 *em, void *stream);
/* device address of the loop's termination flag (int, non-zero once done):
 * a sharded driver reads it asynchronously into pinned memory between
 * replays of its captured pass -> all-reduce -> solve chunks */
int fr_em64_done_ptr(fr_em64 *em, int **d_done);
int fr_em64_sums(fr_em64 *em, double **d_sums, int *width);
/* CTAs and threads per CTA of the grid-resident kernel (launch accounting) */
int fr_em64_launch_info(const fr_em64 *em, int *grid, int *block);
int fr_em64_status(fr_em64 *em, int *done, int *iterations, int *termination, void *stream);
int fr_em64_result(fr_em64 *em, double *R, double *t, double *objectives, double *twist_norms,
                   double *inlier_masses, int *iterations, int *termination, void *stream);

/* ---- float64 device-resident rigid point-to-plane EM loop (pipeline.py:
 * 125-181, residual_mode "point_to_plane"; mstep.py:39-98, 179-210, 421-459)
 * d_ref: float64 planes of m model points (Morton order); the lattice holds
 * the [1, y, n] columns (7; fr_lattice_splat_points64 with FR_VALUES_NORMALS)
 * and its dense float64 grid.  One cooperative launch per fr_em64pl_run: per
 * iteration the E pass (moments, averaged normals, the residual spec stored
 * per point, H and g), the damped 6x6 Cholesky with tenfold escalation, step
 * halving with candidate objectives evaluated over the stored spec (batches
 * of candidate poses built in parallel), max_gn_iters > 1 re-assembly at the
 * accepted pose, update magnitude and termination -- no host round trip.
 * Same result conventions as fr_em64 (cfg->sigma_inv is unused: plane rows
 * and the point rows of invalid normals are unscaled, mstep.py:86-98). */
typedef struct fr_em64pl fr_em64pl;

int fr_em64pl_create(const fr_lattice *lat, const double *d_ref, int64_t m,
                     const fr_rigid_em_config *cfg, void *stream, fr_em64pl **out);
int fr_em64pl_destroy(fr_em64pl *em);
int fr_em64pl_run(fr_em64pl *em, int n_iters, void *stream);
int fr_em64pl_sums(fr_em64pl *em, double **d_sums, int *width);
int fr_em64pl_launch_info(const fr_em64pl *em, int *grid, int *block);
int fr_em64pl_status(fr_em64pl *em, int *done, int *iterations, int *termination, void *stream);
int fr_em64pl_result(fr_em64pl *em, double *R, double *t, double *objectives,
                     double *twist_norms, double *inlier_masses, int *iterations,
                     int *termination, void *stream);

/* ---- device-resident articulated EM loop (pipeline.py:125-181 with an
 * ArticulatedTree, point_to_point; mstep.py:213-229, 348-369, 421-459;
 * kinematics.py:76-229) -------------------------------------------------
 * The tree as plain arrays (host memory): parent index per body (-1 for the
 * root), joint kind (0 fixed, 1 revolute, 2 prismatic), movable slot (joint
 * value index, -1 for fixed), unit joint axis, parent-to-joint frame, and the
 * body-frame centre of the body's points.  At most 32 bodies, 40 parameters.
 * The body-sorted float32 planes and the chunk tables are those of
 * fr_body_pass.  Per iteration (CUDA graph, no host round trip): the body
 * pass over device-resident pass constants, per-body sums, then one CTA
 * runs the M step -- per-body normal equations, forward kinematics, the
 * projected (6 + joints)^2 system, damped Cholesky with tenfold escalation,
 * closed-form halving candidates, extra GN iterations, update magnitude,
 * termination and the next pass constants. */
typedef struct fr_art_tree_desc {
    int n_bodies, n_params, floating;
    const int32_t *parent, *kind, *slot;
    const double *axis, *frame_R, *frame_t, *c_body;
} fr_art_tree_desc;
typedef struct fr_art_em fr_art_em;

/* the device pass of the loop: per-body statistics at device-resident pass
 * constants (d_bodies), no-op once *d_done is set */
int fr_body_pass_dev(const fr_lattice *lat, const float *d_ref, int64_t m, const void *d_bodies,
                     int n_bodies, const int32_t *d_chunk_body, const int64_t *d_chunk_beg,
                     int n_chunks, const int32_t *d_body_chunks, int flags, double *d_sums,
                     double *d_scratch, const int32_t *d_done, void *stream);
int fr_art_em_create(const fr_lattice *lat, const float *d_ref, int64_t m,
                     const fr_art_tree_desc *tree, const double *q0, const double *base_R0,
                     const double *base_t0, const double *body_R0, const double *body_t0,
                     const int32_t *d_chunk_body, const int64_t *d_chunk_beg, int n_chunks,
                     const int32_t *d_body_chunks, const fr_rigid_em_config *cfg, void *stream,
                     fr_art_em **out);
int fr_art_em_destroy(fr_art_em *em);
int fr_art_em_run(fr_art_em *em, void *stream);
/* q: >= 40 doubles (joint values in slot order) */
int fr_art_em_result(fr_art_em *em, double *q, double *base_R, double *base_t,
                     double *objectives, double *twist_norms, double *inlier_masses,
                     int *iterations, int *termination, void *stream);

/* ---- device-resident node-graph EM loop (pipeline.py:125-181 with a
 * NodeGraph; mstep.py:232-369, 421-459; kinematics.py:254-346) -----------
 * Inputs as fr_graph_pass / fr_graph_blocks (input-order float32 planes,
 * skinning, gather lists and the co-skinned pair list pair_lo < pair_hi),
 * plus the node positions, the ARAP edges, a bandwidth-reducing node order
 * `pos` (node -> band position) with block bandwidth bw, per band slot
 * (position i, offset d = 0..bw; slot i * (bw + 1) + d) the contribution
 * list slot_ent[slot_ptr[s] .. slot_ptr[s + 1]) = (kind << 30) | index
 * (kind 0: pair, 1: edge), per node its incident edges
 * inc_ent[inc_ptr[v] ..] = edge << 1 | role (0: k, 1: l), and the initial
 * node poses / dual quaternions.  Per iteration one CUDA graph: E pass and
 * data blocks, the banded system with the ARAP term, block-banded Cholesky
 * with the reference's damping escalation (the SuperLU solve of
 * mstep.py:317-345), all halving candidates in one objective pass, the
 * first accepted step, extra GN iterations under the stored spec, update
 * magnitude and termination.  max_halvings <= 15, max_gn_iters <= 8.
 * Termination 4 of fr_ng_em_result: a dual-quaternion blend degenerated. */
typedef struct fr_ng_em fr_ng_em;

int fr_ng_em_create(const fr_lattice *lat, const float *d_ref, int64_t m, const int32_t *d_sidx,
                    const double *d_swt, int K, int n_nodes, const double *node_pos,
                    const int32_t *edges, int n_edges, const int32_t *d_dptr,
                    const int32_t *d_dent, const int32_t *d_pptr, const int32_t *d_pent,
                    int n_pairs, const int32_t *pair_lo, const int32_t *pair_hi,
                    const int32_t *pos, int bw, const int32_t *slot_ptr,
                    const int32_t *slot_ent, int n_slot_ent, const int32_t *inc_ptr,
                    const int32_t *inc_ent, const double *node_R, const double *node_t,
                    const double *node_dq, int mode, double lambda_reg,
                    const fr_rigid_em_config *cfg, void *stream, fr_ng_em **out);
int fr_ng_em_destroy(fr_ng_em *em);
int fr_ng_em_run(fr_ng_em *em, void *stream);
int fr_ng_em_result(fr_ng_em *em, double *node_R, double *node_t, double *objectives,
                    double *twist_norms, double *inlier_masses, int *iterations,
                    int *termination, void *stream);

/* float64 counterparts of the point helpers above: (n, 3) host rows ->
 * (3, n) float64 device planes (a transpose, no rounding); splat of
 * [1, y, (|y|^2), (n)] from float64 planes; Morton reorder of float64 planes */
int fr_upload_points64(const double *host_xyz, int64_t n, double *d_soa, void *stream);
/* (n, 3) float64 host rows -> (3, n) float64 device planes: a few threads copy the
 * rows into pinned slots, the DMAs land in d_rows (3 n doubles, device scratch),
 * one kernel transposes them into d_soa -- all stream-ordered on `stream`
 * (geometry.py:109-139 PointCloud -> device; no rounding). */
int fr_upload_rows64(const double *host_xyz, int64_t n, double *d_rows, double *d_soa,
                     void *stream);
/* coordinate sums [0:3], minima [3:6], maxima [6:9] of (3, n) float64 planes into
 * d_out (device, 9 doubles), fixed reduction order; d_work: fr_point_stats64_work_doubles()
 * doubles (the model cloud's centre and bounding box, pipeline.py / estep.py:97-112) */
int fr_point_stats64_work_doubles(void);
int fr_point_stats64(const double *d_soa, int64_t n, double *d_work, double *d_out, void *stream);
int fr_lattice_splat_points64(fr_lattice *lat, const double *d_pos, const double *d_normals,
                              int64_t n, int value_mode, void *stream);
int fr_sort_points_morton64(double *d_pos, int64_t n, int planes, int32_t *d_perm, void *stream);
/* Cells of the dense float64 slice grid fr_em64 slices (0: none -- the site
 * box exceeds FR_DENSE64_MAX_CELLS, default 8M cells of 128 B). */
int fr_lattice_dense_cells64(const fr_lattice *lat, int64_t *cells);

#ifdef __cplusplus
}
#endif
#endif /* FILTERREG_B200_H */
