/*
 * rw.h -- C ABI of librw: the B200 (sm_100a) hot path of the hierarchical random walker
 * of Drees, Eilers & Jiang, arXiv 2103.09564 ("PAPER.md").
 *
 * Citations: P:n = PAPER.md line n.  Readings c1..c17 are R1..R17 of
 * DESIGN.md section 3, which adds R19..R29.
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - Pointers named "device" are CUDA device pointers owned by the caller (e.g. torch
 *    tensors).  Host pointers are marked "host".  The library never frees caller memory
 *    and allocates no device memory inside rw_* compute calls (the only library-owned
 *    memory is the rw_queue ring, allocated in rw_queue_create).
 *  - Layout: x fastest, then y, z, then brick, then right-hand side:
 *        idx = ((r*batch + b)*nz + z)*ny*nx + y*nx + x
 *    Brick dims are constant over a batch.  nx must be a multiple of 4; every dim >= 1.
 *    Device pointers must be 16-byte aligned.
 *  - Work is enqueued on the given stream (cudaStream_t passed as void*; NULL = legacy
 *    default stream); results are valid once that stream has synchronised.
 *  - Validation happens before anything is enqueued: on RW_EINVAL nothing ran.
 *  - On any non-OK status rw_last_error() returns a thread-local description.
 */
#ifndef RW_H_
#define RW_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t rw_status;
enum {
  RW_OK = 0,
  RW_EINVAL = 1,        /* bad argument; nothing enqueued                                 */
  RW_ECUDA = 2,         /* a CUDA call failed; rw_last_error() carries the CUDA message     */
  RW_ENOMEM = 3,        /* workspace too small / pinned allocation failed                  */
  RW_EUNSUPPORTED = 4   /* valid request this build does not implement                     */
};

typedef int32_t rw_dtype;
enum { RW_U8 = 0, RW_U16 = 1, RW_I16 = 2, RW_F32 = 3 };

typedef struct { int32_t nx, ny, nz; } rw_dims;
/* Intensity normalisation g = clamp(v*scale + offset, 0, 1) in fp32 (reading c2):
 * u8 {1/255, 0}, u16 {1/65535, 0}, i16 HU window {1/2000, 0.5}, f32 {1, 0}.            */
typedef struct { float scale, offset; } rw_norm;

/* Per-(rhs, brick) exit status written to the optional `status` outputs. */
enum {
  RW_ST_CONVERGED = 1,  /* stopping rule met                                               */
  RW_ST_MAXITER = 2,    /* max_iter reached first (not an error, SURVEY S:208)              */
  RW_ST_TRIVIAL = 3,    /* no fixed voxel (x = x0) or no unknown voxel: 0 iterations       */
  RW_ST_ZERO_B = 4,     /* b = 0 with fixed voxels: exact solution x_U = 0, 0 iterations   */
  RW_ST_BREAKDOWN = 5   /* p.Ap <= 0 or non-finite: brick frozen at its last iterate      */
};

const char* rw_last_error(void);
const char* rw_version(void);

/* ------------------------------------------------------------------------------------
 * rw_brick_weights -- edge weights of the 6-connected brick graph.
 *   P:75 "a 3D grid of vertices with edges between 6-neighbors"; P:77 Grady weight
 *   w_pq = exp(-beta (n[p]-n[q])^2), plus eps > 0 (reading c1) so L_UU is SPD.
 *   vol    device [batch][nz][ny][nx] of `dtype`, normalised with `nm`.
 *   W      device fp32 [3][batch][nz][ny][nx]:  W[a][v] = w(v, v + e_a), a = x,y,z;
 *          0 where v + e_a lies outside the brick (no edges leave a brick, reading c4).
 *   dinv   device fp32 [batch][n] or NULL: 1 / sum of the 6 incident weights (the Jacobi
 *          preconditioner), 0 where fixed[v] != 0.
 *   fixed  device u8 [batch][n] or NULL (NULL: no voxel fixed).
 *   Errors: RW_EINVAL for bad dims/dtype, beta < 0, eps <= 0, NULL vol/W.
 * ---------------------------------------------------------------------------------- */
rw_status rw_brick_weights(const void* vol, rw_dtype dtype, rw_norm nm, int32_t batch,
                           rw_dims d, float beta, float eps, float* W, float* dinv,
                           const uint8_t* fixed, void* stream);

/* ------------------------------------------------------------------------------------
 * rw_brick_weights_ex -- the paper's alternative edge-weight functions,
 *   same output layout and eps floor as rw_brick_weights; pass W to rw_solve_bricks /
 *   rw_solve_labels to solve with them.  Readings R19-R21:
 *   RW_W_GRADY    P:77   w = exp(-beta (g_p - g_q)^2) + eps   (== rw_brick_weights)
 *   RW_W_POISSON  P:133  w = exp(-1/2 (sqrt(n_p) - sqrt(n_q))^2) + eps, n = raw value *
 *                        count_scale clipped at 0 (the normalisation nm is not applied)
 *   RW_W_GAUSSIAN P:127  sigma^2 = mean of (g_p - g_q)^2 over the brick's edges (floored
 *                        1e-8); w = exp(-(g_p - g_q)^2 / (2 sigma^2)) + eps
 *   RW_W_TTEST    P:123-125  Welch t of the (2 radius + 1)^3 neighbourhoods of p and q
 *                        (clipped at the brick border; unbiased variances floored 1e-8);
 *                        w = erfc(|t| / sqrt 2) + eps (two-tailed normal P-value)
 *   workspace  device, >= rw_weights_workspace_bytes(batch, d, spec) bytes (0 for GRADY /
 *              POISSON; batch doubles for GAUSSIAN; 2 fp32 per voxel for TTEST); may be
 *              NULL when that is 0.  Other arguments as rw_brick_weights.
 *   Errors: RW_EINVAL for bad kind, eps <= 0, radius < 1 (TTEST), count_scale <= 0
 *   (POISSON), beta < 0 (GRADY), NULL vol/W, short workspace.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  int32_t kind;        /* RW_W_*                                                         */
  float beta;          /* GRADY                                                          */
  float eps;           /* additive floor, all kinds (reading c1)                          */
  float count_scale;   /* POISSON: counts per raw intensity unit                          */
  int32_t radius;      /* TTEST: neighbourhood radius (1 = 3^3)                           */
} rw_weight_spec;
enum { RW_W_GRADY = 0, RW_W_POISSON = 1, RW_W_GAUSSIAN = 2, RW_W_TTEST = 3 };
size_t rw_weights_workspace_bytes(int32_t batch, rw_dims d, rw_weight_spec spec);
rw_status rw_brick_weights_ex(const void* vol, rw_dtype dtype, rw_norm nm, int32_t batch,
                              rw_dims d, rw_weight_spec spec, float* W, float* dinv,
                              const uint8_t* fixed, void* workspace, size_t ws_bytes,
                              void* stream);

/* ------------------------------------------------------------------------------------
 * rw_solve_workspace_bytes -- device workspace needed by rw_solve_bricks /
 * rw_solve_labels for this shape.  weights_given != 0: the caller passes W (the
 * workspace then holds no weight planes).
 * ---------------------------------------------------------------------------------- */
size_t rw_solve_workspace_bytes(int32_t batch, rw_dims d, int32_t nrhs, int32_t weights_given);

/* ------------------------------------------------------------------------------------
 * rw_solve_bricks -- batched random walker solve (the hot path).
 *   For every brick b and right-hand side r, with S = {v : fixed[b][v] != 0} (seeds and
 *   Dirichlet faces) and U its complement, solves the discrete Dirichlet problem of P:77
 *        L_UU x_U = -B^T x_S,        x_S = values[r][b][S]
 *   with Jacobi-preconditioned CG, matrix-free: the SpMV is the edge-difference
 *   stencil q_i = sum_j w_ij (p_i - p_j) (reading c8), fp32 vectors, fp64 dot products.
 *   All right-hand sides share one operator (W is read once per iteration for all r).
 *   Stopping (reading c5), checked before every iteration on the recurrence residual:
 *        tol_mode 0: ||r_k||_2 <= tol * ||b||_2      tol_mode 1: ||r_k||_2 <= tol
 *   or k == max_iter.  Converged (rhs, brick) pairs drop out of the batch.
 *
 *   batch, d     brick count and brick dims (nx % 4 == 0).
 *   vol, dtype, nm   device intensities (as rw_brick_weights) -- or NULL when W is given.
 *   W            device fp32 [3][batch][n] precomputed weights, or NULL when vol is given.
 *                Exactly one of vol / W must be non-NULL.
 *   fixed        device u8 [batch][n]: 0 = unknown, else Dirichlet.
 *   values       device fp32 [nrhs][batch][n]: Dirichlet values (read only where fixed).
 *   nrhs         1 .. 64 right-hand sides.
 *   beta, eps    weight parameters (used only with vol).  eps > 0.
 *   tol, max_iter, tol_mode   stopping rule; tol > 0, max_iter >= 1.
 *   x0           device fp32 [nrhs][batch][n] initial guess or NULL (0.5 on U, reading c6).
 *   workspace    device, >= rw_solve_workspace_bytes(batch, d, nrhs, W != NULL) bytes,
 *                256-byte aligned; contents are scratch.
 *   prob   out   device fp32 [nrhs][batch][n]: x clamped to [0,1] (reading c9), fixed
 *                voxels hold their values.  Also used as the iterate storage.
 *   iters  out   device int32 [nrhs][batch]: CG iterations (SpMVs) per pair.
 *   resid  out   device fp32 [nrhs][batch] or NULL: recurrence residual at exit,
 *                ||r||/||b|| (mode 0) or ||r|| (mode 1) (reading c16).
 *   status out   device int32 [nrhs][batch] or NULL: RW_ST_* per pair.
 *   labels out   device u8 [batch][n] or NULL: prob[0] > 0.5 (0.5 -> 0, c10).
 *   Not errors: non-convergence (iters = max_iter, status MAXITER); a brick without fixed
 *   voxels (prob = x0 clamped, iters 0, status TRIVIAL).
 *   Stream-ordered and asynchronous: all work is enqueued on `stream` and the call returns
 *   without waiting for it (resident solver: one kernel; streaming solver: one CUDA graph
 *   whose WHILE node runs the iterations on the device, RW_OPT_DEVICE_LOOP).  Outputs are
 *   valid once `stream` reaches this point.  Exceptions that block the host until the loop
 *   has been enqueued: RW_OPT_DEVICE_LOOP = 0, RW_OPT_STREAM_PASSES = 2, residual
 *   replacement, and RW_OPT_COSCHED when it applies.
 * ---------------------------------------------------------------------------------- */
rw_status rw_solve_bricks(int32_t batch, rw_dims d, const void* vol, rw_dtype dtype,
                          rw_norm nm, const float* W, const uint8_t* fixed,
                          const float* values, int32_t nrhs, float beta, float eps,
                          float tol, int32_t max_iter, int32_t tol_mode, const float* x0,
                          void* workspace, size_t ws_bytes, float* prob, int32_t* iters,
                          float* resid, int32_t* status, uint8_t* labels, void* stream);

/* ------------------------------------------------------------------------------------
 * rw_solve_bricks_host -- rw_solve_bricks (nrhs = 1, weights from vol) on HOST buffers with
 *   the transfers pipelined against the solve ("H2D on a copy stream
 *   overlaps compute on the compute stream (events). Results go D2H"; P:105 brick-wise
 *   loading).  The batch is cut into chunks of `chunk` bricks (0: batch/32 rounded up).
 *   Resident-solver shapes (64^3 / 40^3 / 32^3 bricks, u16 or f32 intensities, solver not
 *   forced to streaming): ONE persistent resident launch (plus the L2 worker clusters) covers
 *   the whole batch while the chunks stream through a device ring of min(nchunks, 16) chunk
 *   slots: the H2D copy stream writes chunk c's inputs and then a 4-byte ready flag, the
 *   clusters start a brick of chunk c only once that flag is set, the chunk's last finished
 *   brick sets a host-mapped flag and the calling thread then queues the chunk's D2H copy; a
 *   slot is refilled once the D2H of its previous chunk has run.  Other shapes: chunk c+2's
 *   inputs go host->device on a copy stream while chunk c is solved (separate launches on
 *   two alternating compute streams and workspaces) and chunk c-1's results go
 *   device->host.  Device memory is O(ring) / O(chunk), plus per-brick scalars of the batch.
 *   Library-owned host memory: a per-thread, per-device host-mapped array of chunk-done
 *   flags (4 B per chunk, grown as needed, kept across calls) and one pinned int.  A tool
 *   that serialises launches (CUDA_INJECTION64_PATH set, CUDA_LAUNCH_BLOCKING=1) gets the
 *   chunked pipeline; a persistent launch whose inputs do not arrive within 2 s leaves and
 *   the call redoes the batch on the chunked pipeline (same results).
 *   vol_h, fixed_h, values_h   host [batch][n] (page-locked for overlap; pageable works).
 *   prob_h / labels_h          out host fp32 / u8 [batch][n], either may be NULL.
 *   iters_h out host int32 [batch];  resid_h, status_h  out host [batch] or NULL.
 *   workspace  device, >= rw_solve_host_workspace_bytes(batch, d, dtype, chunk).
 *   Results are identical to rw_solve_bricks on the same bricks (every brick is solved
 *   independently, fixed-order reductions).  The call blocks until the outputs are in host
 *   memory; `stream` is waited on at entry and waits for the call's work at exit.
 *   Errors: as rw_solve_bricks; RW_EINVAL for chunk < 0.
 * ---------------------------------------------------------------------------------- */
size_t rw_solve_host_workspace_bytes(int32_t batch, rw_dims d, rw_dtype dtype, int32_t chunk);
rw_status rw_solve_bricks_host(int32_t batch, rw_dims d, const void* vol_h, rw_dtype dtype,
                               rw_norm nm, const uint8_t* fixed_h, const float* values_h,
                               float beta, float eps, float tol, int32_t max_iter,
                               int32_t tol_mode, int32_t chunk, void* workspace, size_t ws_bytes,
                               float* prob_h, uint8_t* labels_h, int32_t* iters_h,
                               float* resid_h, int32_t* status_h, void* stream);

/* ------------------------------------------------------------------------------------
 * rw_solve_labels -- multi-class random walker, P:79 / P:107: class k's probability is the
 *   solution with class-k seeds = 1 and all other seeds = 0; class = argmax.  Classes are
 *   1..K (K in 2..65); classes 1..K-1 are solved as K-1 right-hand sides sharing one
 *   operator and class K is derived as 1 - sum (linearity of the Dirichlet problem,
 *   reading c11).
 *   seeds    device u8 [batch][n]: 0 = unseeded, k in 1..K = seed of class k.
 *   prob     out device fp32 [K-1][batch][n] (classes 1..K-1, clamped).
 *   labels   out device u8 [batch][n]: argmax over the K probabilities (ties -> lowest
 *            class id), seeds keep their class.
 *   workspace: rw_solve_labels_workspace_bytes(batch, d, K, W != NULL).
 *   Other arguments as rw_solve_bricks.
 * ---------------------------------------------------------------------------------- */
size_t rw_solve_labels_workspace_bytes(int32_t batch, rw_dims d, int32_t K, int32_t weights_given);
rw_status rw_solve_labels(int32_t batch, rw_dims d, const void* vol, rw_dtype dtype,
                          rw_norm nm, const float* W, const uint8_t* seeds, int32_t K,
                          float beta, float eps, float tol, int32_t max_iter,
                          int32_t tol_mode, void* workspace, size_t ws_bytes, float* prob,
                          int32_t* iters, float* resid, uint8_t* labels, void* stream);

/* ------------------------------------------------------------------------------------
 * rw_build_pyramid -- LOD pyramid levels 1..levels of a volume ("applying a 2^3
 *   mean filter and downsampling"; P:109 border bricks smaller than s^3).  Reading c12:
 *   level l+1 voxel (X,Y,Z) = mean of the present level-l children (2X..2X+1, ...);
 *   dims ceil(d/2); integer dtypes: round-half-up floor((sum + floor(cnt/2))/cnt),
 *   bit-exact; f32: fp32 sum in fixed pairwise order, one IEEE division by cnt.
 *   vol        device [d.nz][d.ny][d.nx] of dtype (any dims >= 1; nx need not be % 4).
 *   levels     1..16.
 *   level_out  host array of `levels` device pointers; level l (1-based) has dims
 *              ceil(d / 2^l) applied per level and the input dtype.
 * rw_build_pyramid_slab -- the same over a z-slab [z0, z0+nzs) of a larger volume whose
 *   full dims are `d` (streamed input, config 5): z0 must be a multiple of 2^levels and
 *   nzs a multiple of 2^levels unless z0+nzs == d.nz.  Writes only the output planes
 *   that the slab fully determines; successive slabs produce the same bytes as one call.
 * ---------------------------------------------------------------------------------- */
rw_status rw_build_pyramid(const void* vol, rw_dtype dtype, rw_dims d, int32_t levels,
                           void* const* level_out, void* stream);
rw_status rw_build_pyramid_slab(const void* slab, rw_dtype dtype, rw_dims d, int32_t z0,
                                int32_t nzs, int32_t levels, void* const* level_out,
                                void* stream);

/* ------------------------------------------------------------------------------------
 * rw_hier_segment -- the hierarchical random walker (Eq. 1-4,
 *   H_p pruning).  Readings R22-R26.  Input: a cubic volume of side
 *   D = s 2^k ("we assume a cubical volume size that is a power of two and a
 *   multiple of s") and rasterised labels at full resolution (0 unseeded, 1 foreground,
 *   2 background).  The LOD pyramid (rw_build_pyramid) gives levels 0..k (k = root, one
 *   brick).  The root is solved whole (Eq. 1); then, level by level, every brick whose
 *   parent was not prunable is expanded to a window of side s_e = floor(e s) (Eq. 3),
 *   seeded with its user seeds plus continuous seeds sampled (trilinear) from the parent
 *   level's probability field on window faces interior to the volume (Eq. 2), initialised
 *   from that field, and all such windows of a level are solved as one batch with
 *   rw_solve_bricks (resident solver when s_e is 32, 40 or 64).  The brick's s^3 of each
 *   window solution goes into the level's field; prunable = (hom: max-min < t_hom or
 *   dt: min-0.5 > t_bin or 0.5-max > t_bin) and no seed conflict in the brick;
 *   children of prunable bricks keep the upsampled parent field.
 *   vol      device [D][D][D] of dtype;  seeds  device u8 [D][D][D].
 *   prob     out device fp32 [D][D][D]: the full-resolution foreground probability.
 *   stats    out host (nullable): per level (index = level, 0 = full resolution)
 *            active / solved / pruned_hom / pruned_dt / conflict brick counts, CG iterations.
 *   workspace  device, >= rw_hier_workspace_bytes(d, dtype, cfg).
 *   The call blocks the host (brick lists are built on the host between levels).
 *   Incremental labelling H_it (cfg.incremental = 1, reading R27): with the previous run's
 *   workspace and prob passed back unchanged and the new labels in `seeds`, every solved
 *   brick whose previous node was computed, whose solution moved by less than t_inc over
 *   its s^3 and that has no seed conflict involving a changed label keeps its previous
 *   values and its previous subtree (not descended); recomputed windows start from the
 *   previous solution.
 *   Errors: RW_EINVAL for a non-cubic volume, D != s 2^k, s % 4 != 0, s_e % 4 != 0,
 *   e not in (1, 2], other bad arguments as rw_solve_bricks.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  int32_t s;            /* brick side, level voxels (P:105 suggests 32)                   */
  float e;              /* expansion factor in (1, 2] (P:119 suggests 1.25)               */
  float t_hom, t_bin;   /* pruning thresholds (P:143 0.3, P:149 0.01); < 0 disables one  */
  int32_t prune;        /* 0: solve every brick (plain H), 1: H_p                         */
  float beta, eps, tol; /* Grady weight and solver settings (as rw_solve_bricks)          */
  int32_t max_iter, tol_mode;
  int32_t max_batch;    /* windows per rw_solve_bricks call (workspace size)             */
  int32_t incremental;  /* 1: H_it -- workspace and prob must hold the previous */
                        /*    run on the same volume and geometry; updated in place        */
  float t_inc;          /* reuse threshold max |new - old| (0.01)                    */
} rw_hier_config;
typedef struct {
  int32_t levels;
  int64_t active[16], solved[16], pruned_hom[16], pruned_dt[16], conflict[16], reused[16],
      iters[16];
  int64_t pool_used;    /* rw_hier_segment_ooc: brick-pool slots used (0 otherwise)        */
  double ms_pyramid, ms_levels, ms_output;   /* rw_hier_segment_ooc: host wall time of the    */
                        /* pyramid streaming, the level loop and the output slabs        */
} rw_hier_stats;
size_t rw_hier_workspace_bytes(rw_dims d, rw_dtype dtype, rw_hier_config cfg);
rw_status rw_hier_segment(const void* vol, rw_dtype dtype, rw_norm nm, rw_dims d,
                          const uint8_t* seeds, rw_hier_config cfg, void* workspace,
                          size_t ws_bytes, float* prob, rw_hier_stats* stats, void* stream);

/* ------------------------------------------------------------------------------------
 * rw_hier_segment_ooc -- the hierarchical random walker out of core (P:105
 *   "applicable to arbitrarily large out-of-core datasets ... all computations are local to a
 *   single brick or its direct neighborhood"; P:109-111 volumes of any size; P:151 nearest
 *   computed ancestor; P:261 constant memory).  Same method, seeds and pruning as
 *   rw_hier_segment (H and H_p; readings R22-R26) on volumes of ANY dims (reading R31: level
 *   dims ceil(d/2), root = first level with every dim <= s, smaller border bricks, windows of
 *   side min(s_e, d_l) per axis).  On cubic s 2^k volumes the output equals rw_hier_segment's
 *   bit for bit.
 *   Memory: the volume, the labels and the output stay in HOST memory.  The level-0 data is
 *   streamed through the caller's queue (z-slabs once for the pyramid, then one slot per batch
 *   of leaf windows); the device holds pyramid levels >= 1 of the intensities and seed bits
 *   (1/7 of the volume), per-level page tables, a pool of pool_bricks s^3 fp32 bricks (solved
 *   bricks and the unsolved ones a window samples, materialised as the upsample of their
 *   parent level), one batch of windows and one output slab.  The dense field pyramid of
 *   rw_hier_segment is never formed.
 *   vol_h      host [nz][ny][nx] of dtype;  seeds_h  host u8 [nz][ny][nx] (0 / 1 fg / 2 bg).
 *   cfg        as rw_hier_segment; incremental must be 0 (H_it needs rw_hier_segment).
 *   pool_bricks  brick-pool capacity (RW_ENOMEM if the run needs more; stats.pool_used).
 *   q          rw_queue with slot_bytes >= rw_hier_ooc_queue_bytes(d, dtype, cfg), depth >= 2.
 *   prob_h / labels_h   out host fp32 / u8 [nz][ny][nx], either may be NULL (labels: p > 0.5).
 *   workspace  device, >= rw_hier_ooc_workspace_bytes(d, dtype, cfg, pool_bricks), 256-B aligned.
 *   Host buffers may be pageable or page-locked (cudaMallocHost / cudaHostRegister), detected
 *   per pointer: page-locked vol_h + seeds_h are copied to the device without the staging
 *   copy through the queue's host slots, and a page-locked prob_h / labels_h is written by
 *   the copy engine directly (both then run at the PCIe rate).  Results are the same bits.
 *   Seed slabs are uploaded sparsely (non-zero 4 KiB segments only, the rest a device memset).
 *   Blocks the host (brick lists are built on the host between levels); work on `stream`.
 *   Errors: RW_EINVAL for bad arguments (s % 4, floor(e s) % 4, incremental, small queue),
 *   RW_ENOMEM for a small workspace or a full pool.
 * ---------------------------------------------------------------------------------- */
size_t rw_hier_ooc_workspace_bytes(rw_dims d, rw_dtype dtype, rw_hier_config cfg,
                                   int64_t pool_bricks);
size_t rw_hier_ooc_queue_bytes(rw_dims d, rw_dtype dtype, rw_hier_config cfg);
rw_status rw_hier_segment_ooc(const void* vol_h, rw_dtype dtype, rw_norm nm, rw_dims d,
                              const uint8_t* seeds_h, rw_hier_config cfg, int64_t pool_bricks,
                              struct rw_queue* q, void* workspace, size_t ws_bytes, float* prob_h,
                              uint8_t* labels_h, rw_hier_stats* stats, void* stream);

/* ------------------------------------------------------------------------------------
 * rw_hier_segment_labels_ooc -- multi-class hierarchical segmentation out of core (SURVEY
 *   8(f) f1; P:107 one run per class, the class with the largest foreground probability wins;
 *   P:319 homogeneity pruning only; P:105 / P:261 constant device memory).  K complete
 *   rw_hier_segment_ooc runs in one workspace, class k = 1..K as the foreground: the host
 *   class seeds travel through the queue unchanged and become class k's 0 / 1 / 2 seeds on
 *   the device right after each H2D copy; the output slabs of run k are merged on the host
 *   into the running maximum best_h and its class labels_h (strict >, so ties go to the
 *   lowest class id, reading R11).  dt pruning is disabled whatever cfg.t_bin says.  On cubic
 *   s 2^k volumes best_h / labels_h equal rw_hier_segment_labels' best / out_labels bit for
 *   bit.  Class 1's run builds the intensity pyramid; classes 2..K reuse it and stream only
 *   the class seeds for their seed-bit pyramids (the workspace must not be touched in between).
 *   class_seeds_h  host u8 [nz][ny][nx]: 0 unseeded, 1..K class seeds (any other nonzero
 *               value acts as a background seed for every class).
 *   best_h      out host fp32 [nz][ny][nx]: the winning class's probability (non-NULL).
 *   labels_h    out host u8 [nz][ny][nx]: argmax class 1..K (non-NULL).
 *   stats       out host (nullable): K entries, one per class run.
 *   Other arguments, blocking behaviour and errors as rw_hier_segment_ooc; RW_EINVAL for K
 *   outside 2..255 or a NULL output.
 * ---------------------------------------------------------------------------------- */
rw_status rw_hier_segment_labels_ooc(const void* vol_h, rw_dtype dtype, rw_norm nm, rw_dims d,
                                     const uint8_t* class_seeds_h, int32_t K, rw_hier_config cfg,
                                     int64_t pool_bricks, struct rw_queue* q, void* workspace,
                                     size_t ws_bytes, float* best_h, uint8_t* labels_h,
                                     rw_hier_stats* stats, void* stream);

/* ------------------------------------------------------------------------------------
 * rw_hier_segment_labels -- multi-class hierarchical segmentation (P:107
 *   "The method is run once for each class, where only seeds for the current class are
 *   considered foreground and all other seeds as background ... the class of a voxel is
 *   the one that maximizes the foreground probability"; "only homogeneity-based
 *   pruning ... was applied").  K runs of rw_hier_segment's driver, class k = 1..K as the
 *   foreground, with dt pruning disabled whatever cfg.t_bin says; the intensity pyramid is
 *   built once.  After each run a running argmax updates best / out_labels (strict >, so
 *   ties go to the lowest class id, reading R11).
 *   labels      device u8 [D][D][D]: 0 unseeded, 1..K class seeds (any other nonzero value
 *               acts as a background seed for every class).
 *   prob        out device fp32 [K][D][D][D] (nullable unless incremental): class fields.
 *   best        out device fp32 [D][D][D]: the winning class's probability.
 *   out_labels  out device u8 [D][D][D]: argmax class 1..K.
 *   stats       out host (nullable): K entries, one per class run.
 *   workspace   device, >= rw_hier_labels_workspace_bytes(d, dtype, K, cfg): one
 *               rw_hier_segment workspace (K of them when cfg.incremental, each class keeping
 *               its previous run for H_it) plus one fp32 [D]^3 class field.  A workspace of the incremental size
 *               (cfg.incremental = 1 in the size query) is always used per class, so a
 *               first non-incremental run can be followed by incremental ones.
 *   Errors: as rw_hier_segment; RW_EINVAL for K outside 2..255 or incremental with NULL prob.
 * ---------------------------------------------------------------------------------- */
size_t rw_hier_labels_workspace_bytes(rw_dims d, rw_dtype dtype, int32_t K, rw_hier_config cfg);
rw_status rw_hier_segment_labels(const void* vol, rw_dtype dtype, rw_norm nm, rw_dims d,
                                 const uint8_t* labels, int32_t K, rw_hier_config cfg,
                                 void* workspace, size_t ws_bytes, float* prob, float* best,
                                 uint8_t* out_labels, rw_hier_stats* stats, void* stream);

/* ------------------------------------------------------------------------------------
 * Solver selection.  rw_solve_bricks / rw_solve_labels run one of two implementations of
 * the same Jacobi-PCG with the same stopping rule, status codes and outputs:
 *   streaming  -- CG state in HBM, one fused pass per iteration by default (any brick
 *                 shape, any nrhs, see RW_OPT_STREAM_PASSES);
 *   resident   -- one thread-block cluster per brick keeps the whole CG state on chip
 *                 (shared + tensor memory, registers) for all iterations (SURVEY 8(f)
 *                 f2/f4); bricks of 64^3, 40^3 (s_e of P:119) or 32^3, device
 *                 permitting.  nrhs > 1: every (rhs, brick) pair is its own resident
 *                 solve on the brick's operator (pairs drawn rhs-major from one counter),
 *                 bit-identical to nrhs separate single-rhs calls.
 * RW_OPT_SOLVER: RW_SOLVER_AUTO (default: resident when available, else streaming),
 * RW_SOLVER_STREAMING, RW_SOLVER_RESIDENT (a solve it cannot serve returns
 * RW_EUNSUPPORTED).  Process-wide setting; not thread-safe against concurrent solves.
 * RW_OPT_COSCHED: per-mille share (0..500, default 0 = off) of a resident-eligible batch
 * (>= 64 bricks, vol given, nrhs 1) that runs through the streaming passes on a library
 * stream concurrently with the resident clusters, on the SMs the 16-CTA clusters cannot use
 * (the last bricks of the batch; joined back into the caller's stream).  Needs the
 * workspace rw_solve_workspace_bytes reports (a smaller one disables it).  Those bricks'
 * results agree with the resident solver's to the solver tolerance, not bitwise, so a
 * brick's bits then depend on its position in the batch.  Off by default for that reason
 * (measured on B200: 100 per mille = +4.5 % on the 512 x 64^3 batch, larger shares slower;
 * DESIGN.md 5b).
 * RW_OPT_DEVICE_LOOP: 1 (default) = the streaming solver's iteration loop is device-driven:
 * one CUDA graph whose conditional WHILE node repeats {pass A, loop control} on the GPU, so
 * rw_solve_bricks / rw_solve_labels never block the host (fully stream-ordered; one-pass
 * mode without residual replacement).  0 = host-driven loop (the host polls the active-pair
 * count every 8 iterations and blocks until the loop has been enqueued).  Bit-identical.
 * RW_OPT_RESIDUAL_REPLACE: interval (iterations, default 0 = off) at which the streaming
 * solver replaces the recurrence residual by the true residual b - L_UU x computed in fp32
 * (and flushes the lagged x update).  Experimental: the fp32 true residual floors near
 * 1e-5 of ||b||, so tolerances below that are then never met (R5c).
 * RW_OPT_STREAM_PASSES: 1 (default) or 2 HBM passes per streaming CG iteration.  1: pass
 * B (r -= alpha q and its dots) is folded into the next pass A, which also forms q.D r and
 * q.D q so that beta comes from the one-step expansion r'.z' = r.z - 2 alpha q.D r +
 * alpha^2 q.D q of the true r.z of the same pass (38 instead of 46 bytes per voxel and
 * iteration, one launch instead of two); the stop test uses the true ||r_k|| one pass
 * later, so one extra SpMV runs per (rhs, brick).  2: the classical two-pass form.  The
 * residual-replacement option implies 2.  Iteration counts and probabilities agree to the
 * solver tolerance, not bitwise (measured: identical iteration counts on cfg2/3/4; the one
 * pass is 12-41 % faster).
 * RW_OPT_RESIDENT_WIDE: 0 (default) or 1.  40^3 and 32^3 bricks run as 5- / 4-CTA clusters
 * of 8 planes per CTA (throughput: most bricks per GPU at once); 1 selects 10- / 8-CTA
 * clusters of 4 planes (latency: twice the SMs per brick -- a single 32^3 brick solves in
 * 0.55 instead of 0.74 ms).  Within one setting results are batch-invariant; across the
 * two they agree to the solver tolerance.
 * RW_OPT_L2_WORKERS: 1 (default) or 0.  64^3 resident solves from u16 / f32 intensities
 * (nrhs 1, >= 64 bricks): the 16-CTA clusters fit 7 times (112 SMs); 4-CTA "L2 worker"
 * clusters on the remaining SMs draw bricks from the same counter and run the resident
 * kernel's arithmetic operation for operation with the CG state in global memory, so every
 * brick's outputs are bit-identical whichever cluster solved it (batch-invariant).  The
 * workers use the streaming r region of the workspace (rw_solve_workspace_bytes).
 * RW_OPT_STREAM_ZC: 0 (default, automatic) or the streaming solver's z-chunk (planes per
 * CTA column tile, 4..4096).  The chunk fixes the fp64 partial-sum tree, so results are
 * bitwise reproducible for a given chunk; different chunks agree to the solver tolerance.
 * rw_resident_available(d, nrhs): 1 if the resident solver can serve this shape on the
 * current device, else 0.  Results of the two solvers agree to the solver tolerance, not
 * bitwise (different fp64 reduction trees); each is deterministic and batch-invariant.
 * ---------------------------------------------------------------------------------- */
enum { RW_OPT_SOLVER = 0, RW_OPT_COSCHED = 1, RW_OPT_RESIDUAL_REPLACE = 2,
       RW_OPT_STREAM_PASSES = 3, RW_OPT_RESIDENT_WIDE = 4, RW_OPT_DEVICE_LOOP = 5,
       RW_OPT_STREAM_ZC = 6, RW_OPT_L2_WORKERS = 7 };
enum { RW_SOLVER_AUTO = 0, RW_SOLVER_STREAMING = 1, RW_SOLVER_RESIDENT = 2 };
rw_status rw_set_option(int32_t key, int64_t value);
int64_t rw_get_option(int32_t key);
int32_t rw_resident_available(rw_dims d, int32_t nrhs);

/* ------------------------------------------------------------------------------------
 * Pinned, double-buffered host->device queue for inputs larger than HBM (north star item
 * 5; P:105 constant-memory brick-wise loading).  A ring of `depth` (>= 2) slots, each a
 * pinned host buffer plus a device buffer of slot_bytes, allocated once here (library-
 * owned).  push: waits until the slot's previous consumer released it, copies host_src
 * (pageable, host) into the pinned slot with several host threads -- or, when host_src
 * is itself pinned (page-locked), skips that staging copy and must stay valid until the
 * copy completes on copy_stream -- enqueues the H2D copy on copy_stream and returns the
 * device slot pointer and its id.
 * wait: makes compute_stream wait for that slot's copy.  release: records on
 * compute_stream that the slot's consumers are done (slot reusable after that point).
 * Every push must be matched by a release before the ring comes round to its slot again:
 * a push into a slot that was pushed and not yet released returns RW_EINVAL (nothing is
 * enqueued), so at most `depth` slots are in flight.
 * ---------------------------------------------------------------------------------- */
typedef struct rw_queue rw_queue;
rw_status rw_queue_create(size_t slot_bytes, int32_t depth, rw_queue** q);
rw_status rw_queue_push(rw_queue* q, const void* host_src, size_t bytes, void* copy_stream,
                        void** dev_slot, int32_t* slot_id);
rw_status rw_queue_wait(rw_queue* q, int32_t slot_id, void* compute_stream);
rw_status rw_queue_release(rw_queue* q, int32_t slot_id, void* compute_stream);
void rw_queue_destroy(rw_queue* q);

/* ------------------------------------------------------------------------------------
 * Instrumentation.  Every kernel launch made by librw is counted per kernel class
 * (always on, host-side counter).  With rw_profile_enable(1) each launch is additionally
 * bracketed by CUDA events recorded on the stream it is launched on; rw_profile_read
 * synchronises the pending events and returns the summed device time per class.
 * rw_profile_enable(on) also resets both tallies.  Not thread-safe (one solver thread).
 *   launches  out host int64[RW_K_COUNT] or NULL;  ms  out host double[RW_K_COUNT] or NULL.
 * ---------------------------------------------------------------------------------- */
enum { RW_K_WEIGHTS = 0, RW_K_SETUP = 1, RW_K_PASSA = 2, RW_K_PASSB = 3, RW_K_FINALIZE = 4,
       RW_K_PYRAMID = 5, RW_K_OTHER = 6, RW_K_RESIDENT = 7, RW_K_HIER = 8, RW_K_L2RES = 9,
       RW_K_COUNT = 10 };
rw_status rw_profile_enable(int32_t on);
rw_status rw_profile_read(int64_t* launches, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* RW_H_ */
