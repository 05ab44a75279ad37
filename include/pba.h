/*
 * pba.h — C ABI of the B200-native photometric bundle-adjustment hot path.
 *
 * The reference (photoba, pure Python/numpy) has no FFI; its internal seam
 * for this path is `_LevelProblem` (pkg/src/photoba/solver.py:393-460) plus
 * the solve/update lines of `_solve_level_multi` (solver.py:505-537).  Each
 * entry point below replaces one piece of that seam; the comment on each
 * names the reference code it stands in for.  A maintainer binds these with
 * ctypes; the Python package
 * `paper_2303_16878_b200` is exactly such a binding.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Pointers documented as "device" are
 *    CUDA device pointers owned by the caller (torch tensors in the Python
 *    host); the library never frees caller memory and allocates nothing on
 *    the device itself.  "host" pointers are ordinary CPU memory.
 *  - Every call enqueues work on `stream` (a cudaStream_t passed as void*,
 *    NULL = legacy default stream) and returns without synchronising,
 *    except where a function is documented to read back a status word.
 *  - Return 0 on success, otherwise one of PBA_ERR_*; `pba_last_error()`
 *    returns a human-readable message for the calling thread.
 *  - Poses and extrinsics are rows of 12 doubles: rotation row-major (9)
 *    followed by translation (3).  This is Pose.rotation / Pose.translation
 *    (geometry.py:101-122) flattened.
 */
#ifndef PBA_B200_H
#define PBA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBA_OK 0
#define PBA_ERR_ARG 1          /* -> ValueError */
#define PBA_ERR_CUDA 2         /* -> RuntimeError(pba_last_error()) */
#define PBA_ERR_SINGULAR 3     /* -> UnderConstrainedError / LM lambda bump (solver.py:513-522) */
#define PBA_ERR_PERTURBATION 4 /* -> InvalidPerturbationError (geometry.py:208-212) */

#define PBA_PINHOLE 0   /* sensors.py PINHOLE */
#define PBA_SPHERICAL 1 /* sensors.py SPHERICAL */

/* Per-pair record of the linearisation: the reference `_EdgeTerm`
 * (solver.py:343-353) flattened to 92 doubles.
 *   [ 0..20]  H_ii upper triangle, row-major   (sum J_i^T W J_i)
 *   [21..41]  H_jj upper triangle, row-major   (sum J_j^T W J_j)
 *   [42..77]  H_ij full 6x6, row-major         (sum J_i^T W J_j)
 *   [78..83]  b_i                               (sum J_i^T W e)
 *   [84..89]  b_j
 *   [90]      cost  (sum of Huber losses, solver.py:374)
 *   [91]      count (number of valid blocks, exact integer in a double) */
#define PBA_RECORD_DOUBLES 92
#define PBA_REC_HII 0
#define PBA_REC_HJJ 21
#define PBA_REC_HIJ 42
#define PBA_REC_BI 78
#define PBA_REC_BJ 84
#define PBA_REC_COST 90
#define PBA_REC_COUNT 91

/* Per-chunk partial sums written by pba_linearize (scratch for the caller
 * to allocate): Q = sum w q q^T (21, upper), beta = sum q w e (6), cost,
 * count, 3 pad — see csrc/linearize.cu for the q-basis. */
#define PBA_PARTIAL_DOUBLES 32

/* Texel mask bits (also stored in the separate per-pixel mask plane). */
#define PBA_MASK_DEPTH_VALID 1u   /* CueImage.depth_valid        (cues.py:117)     */
#define PBA_MASK_NORMAL_VALID 2u  /* CueImage.normal_valid       (cues.py:120)     */
#define PBA_MASK_SAMP_CORE 4u     /* sampleable_intensity & _depth (cues.py:132-133) */
#define PBA_MASK_SAMP_NORMAL 8u   /* sampleable_normals          (cues.py:134)     */

/* Sensor intrinsics of one pyramid level: `Intrinsics` (sensors.py:31-76). */
typedef struct pba_camera {
  int32_t model; /* PBA_PINHOLE | PBA_SPHERICAL */
  int32_t width;
  int32_t height;
  int32_t _pad;
  double fx, fy, cx, cy;
  double depth_min, depth_max;
} pba_camera; /* 64 bytes */

/* One (frame, level) image resident in HBM. */
typedef struct pba_frame {
  const void* texels;      /* device: texel planes, width*height*pba_texel_bytes() bytes:
                            * 8 planes of 16-byte pairs, pair k of pixel p at
                            * byte 16*(k*width*height + p); pairs: (I, D), (nx, ny),
                            * (nz, mask u32 | pad), (dI/dcol, dI/drow), (dD/..),
                            * (dnx/..), (dny/..), (dnz/..) */
  const uint8_t* mask;     /* device: width*height mask bytes (PBA_MASK_*) */
  const double* ray_table; /* device: per-column/row unprojection table, see pba_ray_table_doubles() */
  pba_camera cam;
} pba_frame; /* 88 bytes */

/* One directed residual pair i -> j: a `_LevelProblem.contexts` entry
 * (solver.py:400-414). */
typedef struct pba_pair {
  int32_t pose_i, pose_j; /* rows of the pose array (reference node positions) */
  int32_t src, dst;       /* slots in the frame table */
  int32_t ext;            /* row of the extrinsics array (SensorExtrinsics.offset) */
  int32_t n_chunks;       /* number of pixel chunks of this pair (filled by pba_plan_chunks) */
  double occ_tol;         /* occlusion tolerance at this level (solver.py:410); +inf disables */
} pba_pair; /* 32 bytes */

/* Robust-kernel and sampling controls: `SolverConfig` (solver.py:56-91). */
typedef struct pba_config {
  double huber_delta[3]; /* intensity, depth, normal */
  double omega[5];       /* [I, D, nx, ny, nz] = omega_diagonal() (solver.py:90-91) */
  int32_t pixel_stride;  /* source pixel stride (solver.py:200-207) */
  int32_t flags;         /* launch hints (PBA_CFG_*); 0 is always valid */
} pba_config;
/* pba_config.flags: some pair samples a pinhole destination image.  Selects
 * the K1 instantiation that prefetches the next tile's destination footprint
 * into L1 for those pairs (measured: faster on pinhole destinations, slower
 * on the spherical scans).  A launch-shape hint only: results are identical
 * with or without it. */
#define PBA_CFG_PINHOLE_DST 1

/* ---- layout queries --------------------------------------------------- */
size_t pba_texel_bytes(void);
/* Number of doubles in a ray table for `cam`: 2*width + 2*height.
 * Pinhole: [ (u-cx)/fx for u<W | unused W | (v-cy)/fy for v<H | unused H ]
 * Spherical: [ cos az_u | sin az_u | cos el_v | sin el_v ]
 * It is filled on the host (unproject, sensors.py:133-154). */
size_t pba_ray_table_doubles(const pba_camera* cam);
/* Library version string. */
const char* pba_version(void);
/* Message of the last failing call on this thread. */
const char* pba_last_error(void);
/* 1 in the bounds-checked build (libpba_b200_checked.so, -DPBA_CHECKED), else 0. */
int32_t pba_build_checked(void);
/* Number of kernels this library has launched in this process (diagnostics;
 * bench.py reports it per timed step). */
uint64_t pba_kernel_launches(void);

/* ---- per-frame preprocessing: CueImage.__post_init__ (cues.py:106-147) --
 * intensity/depth (H*W doubles) and normals (H*W*3 doubles) are device
 * pointers.  Applies the depth clamp, validity masks, neighbour coherence
 * and central-difference gradients and writes the texel image + mask plane.
 * `scratch` must hold pba_build_texels_scratch_bytes(cam) bytes. */
size_t pba_build_texels_scratch_bytes(const pba_camera* cam);
int pba_build_texels(const pba_camera* cam, const double* intensity, const double* depth,
                     const double* normals, void* texels, uint8_t* mask, void* scratch,
                     void* stream);
/* The same for n_frames frames of one camera stored back to back: frame f's
 * intensity / depth at + f*H*W, normals at + 3*f*H*W, texels at
 * + f*H*W*pba_texel_bytes() bytes, mask at + f*H*W, scratch at
 * + f*pba_build_texels_scratch_bytes(cam) bytes (three launches in all
 * instead of three per frame; identical texels). */
int pba_build_texels_batch(const pba_camera* cam, int32_t n_frames, const double* intensity,
                           const double* depth, const double* normals, void* texels,
                           uint8_t* mask, void* scratch, void* stream);

/* ---- linearisation: _LevelProblem.evaluate per-pair part --------------
 * (solver.py:416-426 -> _edge_term :356-390 -> PairContext.evaluate :222-303)
 *
 * Work is split into chunks of consecutive source pixels (of the strided
 * source grid, row-major): `chunk_pixels` of them, or — when at least 8
 * rows fit in chunk_pixels and the grid width is a multiple of 16 — the
 * multiple of 8 whole rows nearest chunk_pixels (K1 walks those in 16 x 8
 * tiles; the per-pair size is re-derived on the device by the same rule).
 * pba_plan_chunks fills pairs[].n_chunks (host) and
 * writes the chunk table (host, 2 int32 per chunk: pair index, first pixel)
 * and the per-pair chunk offsets (host, n_pairs+1 int32).  Returns the chunk
 * count via *n_chunks_out.  Pass chunk_table == NULL to only count. */
int pba_plan_chunks(pba_pair* pairs, int32_t n_pairs, const pba_camera* src_cams,
                    int32_t pixel_stride, int32_t chunk_pixels, int32_t* chunk_table,
                    int32_t* pair_chunk_offsets, int64_t* n_chunks_out);

/* Bytes of the `partials` scratch of pba_linearize: the chunk partials
 * (n_chunks x PBA_PARTIAL_DOUBLES doubles, rounded up to 256 B) followed by
 * one pair setup (the pair's geometry, formed once per pair) per pair. */
size_t pba_linearize_scratch_bytes(int32_t n_pairs, int64_t n_chunks);
/* frames, pairs, chunk_table, pair_chunk_offsets, poses (n_poses x 12),
 * extrinsics (n_ext x 12), partials (pba_linearize_scratch_bytes bytes) and
 * records (n_pairs x 92) are device pointers; cfg is a host pointer.
 * The chunk table's rows may be permuted freely before upload (it is the
 * CTA launch order; each chunk's partials go to slot
 * pair_chunk_offsets[pair] + first / (the pair's chunk size), so records do not
 * change); the Python host tiles it by (source, destination) frame blocks
 * for L2 locality (device.order_chunks).
 * want_jacobians = 0 is the cost-only path of total_error
 * (solver.py:655-670): ok_jac is not applied and only cost/count are
 * produced (the H/b fields are zero). */
int pba_linearize(const pba_frame* frames, const pba_pair* pairs, int32_t n_pairs,
                  const int32_t* chunk_table, int64_t n_chunks, const int32_t* pair_chunk_offsets,
                  int32_t chunk_pixels, const double* poses, const double* extrinsics,
                  const pba_config* cfg, int32_t want_jacobians, double* partials,
                  double* records, void* stream);

/* ---- assembly: _LevelProblem.evaluate dense part (solver.py:428-449) ---
 * Fixed-edge-order sums of per-pair records into the dense normal
 * equations.  The assembly plan is built on the host by pba_plan_assembly:
 *   slot_of_pose[n_poses] (host in): 6x6 slot of each pose, -1 for the gauge
 *   pair_pose_i/j (host in): pose indices per pair (edge order)
 * Outputs (host): diag_ptr[n_free+1], diag_items[2*n_pairs] (pair<<1|side),
 * off_ptr[n_off+1], off_rc[2*n_off] (row slot, col slot), off_items[n_pairs]
 * (pair<<1|transposed).  *n_off_out receives the number of off-diagonal
 * blocks; pass NULL outputs to only count. */
int pba_plan_assembly(const int32_t* slot_of_pose, int32_t n_poses, const int32_t* pair_pose_i,
                      const int32_t* pair_pose_j, int32_t n_pairs, int32_t* diag_ptr,
                      int32_t* diag_items, int32_t* off_ptr, int32_t* off_rc, int32_t* off_items,
                      int32_t* n_off_out);

/* records (device, n_pairs x 92), plan arrays (device), H (device,
 * dim x dim, row-major, dim = 6*n_free), b (device, dim), totals (device,
 * 2 doubles: cost, count summed in edge order). H is fully overwritten. */
int pba_assemble(const double* records, int32_t n_pairs, int32_t n_free, const int32_t* diag_ptr,
                 const int32_t* diag_items, int32_t n_off, const int32_t* off_ptr,
                 const int32_t* off_rc, const int32_t* off_items, double* H, double* b,
                 double* totals, void* stream);
/* The same sums into the block-sparse normal matrix (north_star: "into the
 * block-sparse H/b"; what DeviceLevel uses): Hb (device, n_blocks x 36) holds
 * the 6x6 blocks in the order of the block-row CSR of the damped system's
 * non-zero blocks (row_ptr / cols: the diagonal and both orientations of
 * every off-diagonal block, columns ascending), block e at Hb[36 e + 6 k + l].
 * diag_blk[s] (n_free) and off_blk[2 o], off_blk[2 o + 1] (2 n_off) are the
 * CSR positions of slot s's diagonal block and of the (row, col) / (col, row)
 * blocks of off-diagonal target o (off_rc order of pba_plan_assembly).
 * Every block is written (no clearing pass); per entry the sums run in the
 * same edge order as pba_assemble, so Hb equals the dense H's blocks bit for
 * bit (solver.py:428-449). */
int pba_assemble_bsr(const double* records, int32_t n_pairs, int32_t n_free,
                     const int32_t* diag_ptr, const int32_t* diag_items, int32_t n_off,
                     const int32_t* off_ptr, const int32_t* off_items, const int32_t* diag_blk,
                     const int32_t* off_blk, double* Hb, double* b, double* totals,
                     void* stream);
/* Cost/count only (cost-only path and the LM acceptance test). */
int pba_sum_totals(const double* records, int32_t n_pairs, double* totals, void* stream);

/* ---- linear solve: np.linalg.solve(H + lam*diag(H), -b) (solver.py:510-512)
 * Dense fp64 Cholesky of the damped system on 64x64 tiles.  H, b: device
 * inputs (not modified).  tile_env: optional host array of ceil(dim/64)
 * ints, tile_env[i] = first tile column that may be non-zero in tile row i
 * (the matrix envelope; Cholesky fill-in never leaves it) — NULL means dense.
 * Narrow envelopes over many tiles (chain-like pose graphs) are solved by
 * nested dissection (independent segments batched, separators last); other
 * matrices by the sequential tiled factorisation.
 * work: device, pba_solve_work_bytes(dim) bytes.  delta: device output.
 * status: device int32 written 0 on success, 1 when the damped matrix is
 * not positive definite (the reference's LinAlgError). */
size_t pba_solve_work_bytes(int32_t dim);
int pba_solve_dense(const double* H, const double* b, int32_t dim, double lam,
                    const int32_t* tile_env, void* work, double* delta, int32_t* status,
                    void* stream);
/* Graph-capturable form: lambda read from device memory (lam_dev, one
 * double; NULL -> lam) when the kernels run, and with PBA_SOLVE_REUSE_PLAN
 * the tile tables a previous call with the same dim / tile_env put in
 * `work` are reused instead of copied from the host again — so the call
 * issues only kernel launches and a memset, and a captured LM step replays
 * with a new lambda. */
#define PBA_SOLVE_REUSE_PLAN 1
int pba_solve_dense_ex(const double* H, const double* b, int32_t dim, double lam,
                       const double* lam_dev, const int32_t* tile_env, void* work, int32_t flags,
                       double* delta, int32_t* status, void* stream);
/* The same factorisation reading the block-sparse Hb of pba_assemble_bsr
 * (row_ptr / cols its block-row CSR): the damped envelope tiles are built
 * straight from the blocks, so no dense H exists. */
int pba_solve_dense_bsr(const double* Hb, const int32_t* row_ptr, const int32_t* cols,
                        const double* b, int32_t dim, double lam, const double* lam_dev,
                        const int32_t* tile_env, void* work, int32_t flags, double* delta,
                        int32_t* status, void* stream);

/* ---- the same system by block-Jacobi PCG (App. C c3: "LM with block-Jacobi
 * PCG"); replaces np.linalg.solve at solver.py:510-512 by an iterative solve.
 * One cooperative kernel.  H: the assembled dense matrix (n_free 6x6 block
 * rows, dim = 6 n_free, full symmetric storage as pba_assemble writes it).
 * row_ptr (n_free+1) / cols: device block-row CSR of the structurally
 * non-zero blocks (diagonal included), cols ascending per row.  Stops when
 * ||r|| <= tol ||b|| or after max_iter iterations (the iterate is then
 * returned as an inexact LM step).  work: pba_pcg_work_bytes(n_free) bytes.
 * status: 0 ok, 1 when a damped diagonal block or the system is not
 * positive definite.  info (device, 3 doubles): iterations, final relative
 * residual, converged flag.  The iteration vectors live in registers of
 * co-resident CTAs, so n_free <= 32 x (resident CTAs) (~9,400 poses on a
 * B200); larger systems return PBA_ERR_ARG (use pba_solve_dense). */
size_t pba_pcg_work_bytes(int32_t n_free);
int pba_solve_pcg(const double* H, const double* b, int32_t n_free, double lam,
                  const int32_t* row_ptr, const int32_t* cols, int32_t max_iter, double tol,
                  void* work, double* delta, int32_t* status, double* info, void* stream);
/* The same with lambda read from device memory (lam_dev; NULL -> lam). */
int pba_solve_pcg_ex(const double* H, const double* b, int32_t n_free, double lam,
                     const double* lam_dev, const int32_t* row_ptr, const int32_t* cols,
                     int32_t max_iter, double tol, void* work, double* delta, int32_t* status,
                     double* info, void* stream);
/* PCG on the block-sparse Hb (its CSR is the mat-vec's row_ptr / cols;
 * diag_blk[s] = CSR position of the diagonal block of block row s). */
int pba_solve_pcg_bsr(const double* Hb, const double* b, int32_t n_free, double lam,
                      const double* lam_dev, const int32_t* row_ptr, const int32_t* cols,
                      const int32_t* diag_blk, int32_t max_iter, double tol, void* work,
                      double* delta, int32_t* status, double* info, void* stream);

/* ---- pose update: _LevelProblem.apply_step (solver.py:451-460) --------
 * poses_out[k] = poses_in[k] * exp(delta[slot_k]) for every non-gauge pose
 * (geometry.py:202-219), in fp64.  generation (device int32, n_poses) is
 * Pose.generation; gen_out receives the new counters and rotations are
 * re-orthonormalised when they reach 1000 (geometry.py:17, 137-143).
 * status (device int32) is set to 1 when some ||dq|| >= 1. */
int pba_apply_step(const double* poses_in, const int32_t* gen_in, const double* delta,
                   int32_t n_poses, int32_t gauge, double* poses_out, int32_t* gen_out,
                   int32_t* status, void* stream);

/* ---- device-resident LM level: _solve_level_multi (solver.py:505-537) ----
 * A CUDA graph with a conditional WHILE node runs a whole LM level without a
 * host round trip per iteration.  pba_lm_loop_begin creates the graph and
 * starts capturing `stream` (a non-default stream) into the loop body; the
 * caller then issues one iteration on that stream — the damped solve with
 * lambda read from lam_dev, pba_apply_step into the candidate buffers,
 * pba_linearize + assembly of the candidate, and pba_lm_decide (which also
 * copies the candidate buffers over the current ones on acceptance) — and
 * pba_lm_loop_end instantiates it.  Each pba_lm_loop_launch runs the body until
 * pba_lm_decide clears the loop condition.
 * state: device doubles, PBA_LM_STATE_DOUBLES of them (indices below), set
 * by the host before a launch (iteration = 1, n_records = 0, stop = error =
 * 0) and read back after it.  records: device doubles,
 * PBA_LM_RECORD_DOUBLES per iteration: lambda, cost, count, accepted —
 * solver.py's IterationRecord fields — then the candidate's cost and count.
 * pba_lm_decide applies one iteration's accept / reject, lambda update,
 * termination tests and loop-head test exactly as the reference loop does;
 * a singular first solve or an ||dq|| >= 1 step stops the loop with
 * state[PBA_LM_ERROR] set (the host raises UnderConstrainedError /
 * InvalidPerturbationError). */
#define PBA_LM_COST 0
#define PBA_LM_COUNT 1
#define PBA_LM_LAMBDA 2
#define PBA_LM_FACTOR 3
#define PBA_LM_REL_TOL 4
#define PBA_LM_LAMBDA_CEILING 5
#define PBA_LM_COST_FLOOR 6
#define PBA_LM_ITERATION 7
#define PBA_LM_MAX_ITERATIONS 8
#define PBA_LM_STOP 9
#define PBA_LM_ERROR 10
#define PBA_LM_N_RECORDS 11
#define PBA_LM_ACCEPTED 12
#define PBA_LM_STATE_DOUBLES 16
#define PBA_LM_ERR_UNDERCONSTRAINED 1
#define PBA_LM_ERR_PERTURBATION 2
#define PBA_LM_MAX_COPY 8
#define PBA_LM_RECORD_DOUBLES 6
typedef struct pba_lm_loop pba_lm_loop;
int pba_lm_loop_begin(void* stream, pba_lm_loop** loop, uint64_t* handle);
/* One iteration's decision, then on acceptance dst[k] <- src[k] (the
 * candidate poses / generations / H / b / totals over the current ones;
 * bytes[k] a multiple of 4; device pointers in host arrays of
 * n <= PBA_LM_MAX_COPY). */
int pba_lm_decide(double* state, double* records, const int32_t* status_solve,
                  const int32_t* status_step, const double* new_totals, double* lam_dev,
                  uint64_t handle, void* const* dst, const void* const* src,
                  const int64_t* bytes, int32_t n, void* stream);
int pba_lm_loop_end(pba_lm_loop* loop);
int pba_lm_loop_launch(pba_lm_loop* loop, void* stream);
void pba_lm_loop_destroy(pba_lm_loop* loop);

/* ---- match-graph construction: overlap_ratio (graph.py:70-101) ---------
 * Valid-projection counts for directed candidate pairs (device pointers):
 * points: sensor-frame points of every frame's valid graph-level pixels
 * (3 doubles each, concatenated, built on the host exactly as the
 * reference); point_offsets: n_frames+1; pair_src: source frame per pair;
 * transforms: 12 doubles per pair, the composed sensor_j^-1 * sensor_i;
 * dst_cams: destination camera per pair; counts: int64 per pair.  The host
 * re-decides pairs whose ratio is within a few points of the threshold
 * with the exact path (pairgraph.build_graph). */
int pba_overlap_counts(const double* points, const int64_t* point_offsets, const int32_t* pair_src,
                       const double* transforms, const pba_camera* dst_cams, int32_t n_pairs,
                       double bound_slack, int64_t* counts, void* stream);

/* ---- cue-pyramid builder: build_pyramid (cues.py:342-375) ---------------
 * NormalConfig (cues.py:26-39); min_points is compared as a double like the
 * reference's float window count. */
typedef struct pba_normal_config {
  double k_tau, radius_min, radius_max, min_points, degeneracy_ratio;
} pba_normal_config;

/* Scratch for pba_estimate_normals: the (n, 10, H, W) fp64 moment table. */
size_t pba_normals_scratch_bytes(const pba_camera* cam, int32_t n_frames);
/* estimate_normals (cues.py:187-246) for n_frames depth/range images of one
 * camera (device (n, H, W) fp64, raw: non-finite and out-of-range pixels are
 * invalid) -> observer-facing unit normals (device (n, H, W, 3), zero where
 * no plane fits).  ray_table: pba_ray_table_doubles(cam) doubles (device).
 * Bit-equal to the reference up to the 3x3 eigenproblem (cues.py:239,
 * numpy.linalg.eigh), which is solved by Jacobi; every pixel whose gates
 * or normal could differ under LAPACK is left zero and listed in `recheck`
 * (device, recheck_capacity records of PBA_NORMALS_RECHECK_DOUBLES doubles:
 * [flat pixel index f*H*W + p, S00, S11, S22, S10, S20, S21, x, y, z]) for
 * the caller to decide with eigh; *recheck_count (device int32) receives
 * the number of such pixels (records beyond the capacity are dropped: call
 * again with a larger buffer). */
#define PBA_NORMALS_RECHECK_DOUBLES 10
int pba_estimate_normals(const pba_camera* cam, const double* ray_table, const double* depth,
                         int32_t n_frames, const pba_normal_config* cfg, double* normals,
                         void* scratch, double* recheck, int32_t recheck_capacity,
                         int32_t* recheck_count, void* stream);
/* _downscale_cues (cues.py:278-326) of n_frames full-resolution cue sets
 * (cam = full-resolution camera; depth already cleaned of non-finite values
 * as build_pyramid does) to one level of scale s: out_h/out_w must equal
 * floor(H*s)/floor(W*s).  Bit-equal to the reference. */
int pba_downscale_cues(const pba_camera* cam, double scale, int32_t n_frames,
                       const double* intensity, const double* depth, const double* normals,
                       int32_t out_h, int32_t out_w, double* out_intensity, double* out_depth,
                       double* out_normals, void* stream);

/* ---- dataset rasters: read_intensity / read_depth (dataset_io.py:74-136) --
 * raw: device bytes of PGM P5 payloads (headers stripped by the host),
 * frames back to back; n_samples pixels.  16-bit samples are big-endian.
 * Intensity: raw / 65535 (8-bit: raw / 255); depth: raw * depth_scale
 * (raw 0 = invalid -> 0.0).  out: n_samples doubles (device). */
#define PBA_RASTER_U8_INTENSITY 0
#define PBA_RASTER_U16_INTENSITY 1
#define PBA_RASTER_U16_DEPTH 2
int pba_decode_raster(const uint8_t* raw, int64_t n_samples, int32_t kind, double depth_scale,
                      double* out, void* stream);

/* ---- diagnostics ------------------------------------------------------
 * The table-corrected fp64 atan2 the spherical projection uses
 * (csrc/fastmath.cuh), exposed so tests can bound its error against the
 * library atan2 / numpy.arctan2 (sensors.py:120-121).  Device pointers. */
int pba_atan2_batch(const double* y, const double* x, int64_t n, double* out, void* stream);
/* Section timing of the linearisation kernel (PBA_LIN_VARIANT=24 only):
 * summed clock64 cycles and visit counts of 8 per-pixel sections, host
 * arrays of 8; reset != 0 zeroes the counters after reading. */
int pba_diag_section_cycles(uint64_t* cycles, uint64_t* counts, int32_t reset);
/* Device-resident LM loop timing (diagnostics): out[8 * iteration + slot]
 * = %globaltimer (ns) when the stamp runs; iteration read from the loop
 * state (PBA_LM_ITERATION).  Issued between the captured calls of a loop
 * body it gives per-iteration phase times. */
int pba_diag_lm_stamp(const double* state, int64_t* out, int32_t slot, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PBA_B200_H */
