/*
 * spamm.h — C ABI of the B200 (sm_100a) SpAMM / Newton-Schulz library
 * (libspamm_b200.so).  No C++ or torch types cross this boundary.
 *
 * Method: Challacombe, Haut & Bock, "A N-Body Solver for Square Root
 * Iteration", arXiv 1508.05856 (PAPER.md; citations P:<line>):
 *   - quadtree matrix with Frobenius-norm decorations ............ P:115-129
 *   - SpAMM product a (x)_tau b, Eq. newspamm; cull iff
 *     ||a^i|| ||b^i|| < tau ||a|| ||b|| ............................ P:199-216
 *   - dual-channel Newton-Schulz square-root iteration, Eq.
 *     cannonical, in the north_star form of BASELINE.json:
 *     X = Z (x) Y, H = 1/2(3I - X), Y <- Y (x) H, Z <- H (x) Z ..... P:380-389
 *   - trace error t_k = (n - tr X)/n .............................. P:438-440
 *
 * Conventions (all entry points):
 *   - Return SPAMM_OK (0) or an error code; never throws / exits.  A textual
 *     reason is available from spamm_last_error(ctx) until the next call.
 *   - Work is enqueued on the context's CUDA stream.  Calls that return host
 *     values (spamm_norm, spamm_multiply stats, spamm_ns_sqrt history,
 *     spamm_export_tasks, spamm_mat_info) synchronise that stream.
 *   - "Pointer, host or device": the library inspects the pointer with
 *     cudaPointerGetAttributes; host memory (pageable or pinned) is staged
 *     through the stream, device memory is read in place.
 *   - Matrices are square, n = b * 2^L with b in {16, 32, 64}; dense inputs
 *     are row-major fp64 with leading dimension ld >= n.  A leaf block is
 *     "present" iff its fp64 sum of squares is > 0 (reading L6);
 *     absent blocks are exact zeros and never form leaf tasks.
 *   - spamm_mat handles returned through out-parameters are owned by the
 *     caller and released with spamm_mat_free.  Each matrix holds its context:
 *     spamm_ctx_destroy while matrices are alive only marks the context, and
 *     the teardown happens at the last spamm_mat_free (no other call may use a
 *     destroyed context; freeing its remaining matrices is the one exception).
 *   - All device memory comes from the context allocator (the Python layer
 *     passes PyTorch's caching allocator), else cudaMallocAsync on the stream.
 */
#ifndef SPAMM_B200_H
#define SPAMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spamm_ctx_s *spamm_ctx;
typedef struct spamm_mat_s *spamm_mat;
typedef struct spamm_comm_s *spamm_comm;

typedef enum {
    SPAMM_OK = 0,
    SPAMM_EINVAL = 1,      /* bad argument (negative / non-finite tau, b, iters, NULL) */
    SPAMM_ESHAPE = 2,      /* operands differ in n or b                                 */
    SPAMM_ENOMEM = 3,      /* allocator returned NULL                                   */
    SPAMM_ECUDA = 4,       /* CUDA runtime / launch error                               */
    SPAMM_ENCCL = 5,       /* NCCL unavailable or a collective failed                   */
    SPAMM_ENOTFINITE = 6,  /* non-finite root norm or trace error (history is kept)     */
    SPAMM_ECAPACITY = 7    /* internal capacity could not be grown                      */
} spamm_status;

/* Device allocator callbacks (stream-ordered).  alloc returns NULL on failure. */
typedef struct {
    void *(*alloc)(size_t bytes, void *stream, void *user);
    void (*free)(void *ptr, size_t bytes, void *stream, void *user);
    void *user;
} spamm_allocator;

/* Per-product counters (filled on request; host memory). */
typedef struct {
    int64_t tasks;              /* surviving leaf triples |S| (P:217-218 vol)        */
    int64_t segments;           /* output blocks (i,j) with >= 1 surviving task      */
    int64_t candidates;         /* leaf-level candidate triples tested               */
    int64_t level_survivors[24];/* survivors per quadtree level (index = level)      */
    double flops;               /* 2 b^3 |S|                                         */
    int64_t halo_blocks;        /* row partition: remote right-operand blocks fetched */
    int64_t local_segments;     /* row partition: segments needing no remote block (run
                                   while the halo is exchanged)                        */
    int32_t transport;          /* row partition, world > 1: 1 = halo exchange over the
                                   communicator (v2), 2 = peer memory: remote tiles read in
                                   place from the owners' pools (v3); 0 otherwise        */
} spamm_stats;

/* Options of spamm_ns_sqrt (NULL => defaults).  History buffers are HOST memory. */
typedef struct {
    double tau_s;           /* sensitive threshold for Y (x) H; < 0 => tau */
    double mu;              /* relative Tikhonov shift: Y0 = (s/c + mu I)/(1+mu); 0 => none
                               (reading L13)                       */
    double scale;           /* > 0 => use as c ~ ||s||_2; else power iteration          */
    int32_t power_iters;    /* power steps for c (default 100, reading L12)             */
    double *t_history;      /* [iters] trace errors t_k, nullable                        */
    spamm_stats *per_product;/* [3*iters] stats of X, Y', Z' per k, nullable             */
    double *c_out;          /* scale actually used, nullable                             */
    double t_stop;          /* > 0 => stop after the first k with |t_k| <= t_stop (convergence
                               monitored by the trace error); 0 => run all iters  */
    int32_t *iters_done;    /* number of NS steps actually run, nullable                 */
    int32_t map;            /* 0: H = 1/2 (3I - X) (north_star, alpha = 1, eps = 0);
                               1: scaled + stabilised H = h_alpha[(1-2eps) X + eps I] with the
                               paper's sigmoids alpha(t_k), eps(t_k)             */
} spamm_ns_opts;

/* ---------------------------------------------------------------- context */
/* device: CUDA ordinal; cuda_stream: cudaStream_t (NULL = a library-owned stream);
 * allocator: nullable (=> cudaMallocAsync). */
spamm_status spamm_ctx_create(int device, void *cuda_stream, const spamm_allocator *allocator,
                              spamm_ctx *out);
void spamm_ctx_destroy(spamm_ctx ctx);
const char *spamm_last_error(spamm_ctx ctx);
/* number of library kernels launched on this context since creation */
int64_t spamm_kernel_launches(spamm_ctx ctx);

/* ------------------------------------------------- row-partitioned path */
/* SURVEY.md §8(e) / BASELINE.json north_star ("output block-rows are partitioned
 * over GPUs; NCCL over NVLink all-gathers the operand blocks and norms each shard
 * needs").  Output block rows are independent given (i) the complete leaf-norm
 * arrays of both operands and (ii) the right operand's blocks the local tasks
 * use (Eq. newspamm: C_ij = sum_k A_ik B_kj, k over all rows).  On a
 * context with a communicator:
 *   - every matrix stores only the rank's block rows [r0, r1) (pool, slot map),
 *     while its squared-norm pyramid is complete and bitwise identical on all
 *     ranks (leaf rows all-gathered after every build / product, pyramid summed
 *     in the fixed order of the single-device path);
 *   - spamm_multiply / spamm_ns_step / spamm_ns_sqrt cull only the local output
 *     rows, fetch the remote right-operand blocks their tasks use (request lists
 *     + grouped send/recv of packed blocks), run the leaf GEMM on local segments,
 *     and all-gather the new leaf norms and the trace partials;
 *   - spamm_build_tree* accept the full input (or any superset of the local rows)
 *     and keep the local rows; readers (spamm_to_dense, spamm_export_blocks,
 *     spamm_get_blocks, spamm_export_tasks, spamm_mat_info) see local rows only;
 *     spamm_norm and spamm_level_norms2 are global.
 * Each output block is computed by exactly one rank with the same k-order, so Y
 * and Z are bitwise identical for every world size (tests/test_gpu_dist.py).
 * All ranks must issue the same sequence of calls (SPMD); a failing rank leaves
 * its peers blocked in the next collective. */

/* NCCL unique id (128 opaque bytes) for spamm_comm_nccl_create; rank 0 draws it
 * and the caller broadcasts it (the Python layer uses torch.distributed).  NCCL
 * is loaded with dlopen (the libnccl.so.2 already in the process, else
 * $SPAMM_NCCL_LIB, else the system one).  Errors: ENCCL. */
spamm_status spamm_comm_nccl_unique_id(void *id128);
/* One rank of an NCCL communicator on CUDA device `device` (owned by the
 * returned handle; destroyed by spamm_comm_destroy). */
spamm_status spamm_comm_nccl_create(const void *id128, int32_t rank, int32_t world, int32_t device,
                                    spamm_comm *out);
/* An in-process group of `world` ranks (comms[0..world-1]) for host threads that
 * each drive their own context, on one device or several: collectives are
 * stream-ordered device copies joined by host barriers and CUDA events (no
 * kernel ever waits on another rank's kernel).  The group also offers peer
 * memory: ranks publish their right operand's pool and slot
 * map once per product and the leaf GEMM bulk-copies remote tiles straight from
 * the owner's pool (peer access over NVLink between devices, enabled on first
 * use); no halo is exchanged.  Where two ranks' devices cannot reach each other,
 * or with SPAMM_PEER=0, products use the halo exchange.  The arithmetic is the
 * same on every transport (bitwise equal results). */
spamm_status spamm_comm_local_group(int32_t world, spamm_comm *comms);
void spamm_comm_destroy(spamm_comm comm);
/* Attach a communicator (borrowed; NULL detaches) and the row partition:
 * row_start[world+1] in leaf block rows, ascending, row_start[0] = 0,
 * row_start[world] = nb of every matrix used (host pointer, copied; NULL =>
 * equal split floor(p*nb/world) per matrix).  Matrices created before the
 * call keep their partition.  Errors: EINVAL (bad partition / world). */
spamm_status spamm_ctx_set_comm(spamm_ctx ctx, spamm_comm comm, const int32_t *row_start);
/* Local block-row range [r0, r1) of m on this rank (single device: [0, nb)). */
spamm_status spamm_mat_rows(spamm_mat m, int32_t *r0, int32_t *r1);
/* Per-block-row leaf task counts of A (x)_tau B (rows i of the whole matrix, from
 * the replicated norms only; no GEMM).  counts: [nb] int64, host.  For
 * balancing a row partition on measured work. */
spamm_status spamm_row_task_counts(spamm_ctx ctx, spamm_mat A, spamm_mat B, double tau,
                                   int64_t *counts);

/* ------------------------------------------------------------ quadtree */
/* Build the quadtree of a dense n x n row-major matrix (host or device pointer):
 * leaf norms, Morton-ordered norm pyramid, packed block pool. */
spamm_status spamm_build_tree(spamm_ctx ctx, const double *dense, int64_t n, int64_t ld,
                              int32_t b, spamm_mat *out);
/* Build from a block list: nblocks blocks (bi[t], bj[t]) each b*b row-major at
 * blocks + t*b*b (host or device pointers; coordinates must be distinct). */
spamm_status spamm_build_tree_blocks(spamm_ctx ctx, int64_t n, int32_t b, int64_t nblocks,
                                     const int32_t *bi, const int32_t *bj, const double *blocks,
                                     spamm_mat *out);
void spamm_mat_free(spamm_mat m);
/* n, b, number of stored blocks (syncs). */
spamm_status spamm_mat_info(spamm_mat m, int64_t *n, int32_t *b, int64_t *nblocks);
/* Frobenius norm ||m||_F = sqrt(root of the squared-norm pyramid) (syncs). */
spamm_status spamm_norm(spamm_ctx ctx, spamm_mat m, double *fro);
/* Dense copy (host or device pointer, ld >= n); absent blocks are written as 0. */
spamm_status spamm_to_dense(spamm_ctx ctx, spamm_mat m, double *dense, int64_t ld);
/* Squared Frobenius norms of one pyramid level (0 = root, L = leaves) as a
 * 2^level x 2^level row-major array (host or device pointer). */
spamm_status spamm_level_norms2(spamm_ctx ctx, spamm_mat m, int32_t level, double *out);
/* Gather nreq blocks (bi[t], bj[t]) into out + t*b*b (zeros if absent); present[t]
 * (nullable) = 1/0.  All pointers host or device. */
spamm_status spamm_get_blocks(spamm_ctx ctx, spamm_mat m, int64_t nreq, const int32_t *bi,
                              const int32_t *bj, double *out, int32_t *present);

/* --------------------------------------------------------------- SpAMM */
/* C = A (x)_tau B (Eq. newspamm): level-by-level two-sided norm query
 * keeping (i,k,j) iff n2A[i,k]*n2B[k,j] >= tau^2 ||A||^2 ||B||^2 (squared form of
 * P:205, reading L5), then C_ij = sum_k A_ik B_kj over surviving k (FP64 DMMA).
 * Errors: ESHAPE (n or b differ), EINVAL (tau < 0 or not finite). */
spamm_status spamm_multiply(spamm_ctx ctx, spamm_mat A, spamm_mat B, double tau, spamm_mat *C,
                            spamm_stats *stats /* nullable, host */);
/* C = A^T (x)_tau B: the SpAMM product of the transposed left operand (node (I,K) of
 * A^T is node (K,I) of A; ||a^T|| = ||a||, so A's norms serve as they are).  Needed by
 * the single-channel iteration.  Errors as
 * spamm_multiply, plus EINVAL on a row-partitioned context (A^T's rows are not local). */
spamm_status spamm_multiply_t(spamm_ctx ctx, spamm_mat A, spamm_mat B, double tau, spamm_mat *C,
                              spamm_stats *stats /* nullable, host */);
/* Leaf triples (i,k,j) of the last product on ctx, grouped by output block (i,j)
 * in Morton order, k ascending; ikj is HOST [3*cap]; *n = total count. */
spamm_status spamm_export_tasks(spamm_ctx ctx, int32_t *ikj, int64_t cap, int64_t *n);

/* Product-volume instrumentation (the lensing of P:804-823):
 * histogram of d = max(|i-j|, |i-k|, |j-k|) over the last product's surviving leaf
 * triples (i,k,j); hist: HOST [nbins] int64, d >= nbins-1 counted in the last bin.
 * Exact integer counts.  Synchronises. */
spamm_status spamm_task_distance_hist(spamm_ctx ctx, int64_t *hist, int32_t nbins);

/* Per-product volume recorder: the paper's lensing evidence is
 * per iteration and per product (the y_k and x_k volumes of P:740-745, "Locality"
 * P:804-813; "sparse VTK output for visualization of the ijk product volumes",
 * P:418-419).  While a sink is attached (spamm_ctx_set_volume_sink), EVERY SpAMM
 * product the context runs (spamm_multiply[_t], the three products of each
 * spamm_ns_step / spamm_ns_sqrt iteration in the order X, Y', Z', the single-channel
 * and regularised paths) appends one record, after its cull and before its GEMM:
 *   ntasks[p]            surviving leaf triples of product p;
 *   hist[p*nbins + d]    triples with max(|i-j|, |i-k|, |j-k|) = d (last bin: >= nbins-1),
 *                        when nbins > 0 and hist != NULL;
 *   ikj                  the triples themselves (i,k,j), product after product, in the
 *                        GEMM's order (output block Morton order, k ascending), while
 *                        ikj_count < ikj_cap; ikj_needed counts all of them.
 * Records beyond nprod_cap only advance nprod.  All arrays are HOST memory owned by
 * the caller and must outlive the attachment.  Row partition: each rank records
 * its own rows' triples.  Recording synchronises the stream once per product
 * (instrumentation, not for timed runs).  Errors: EINVAL (nprod_cap < 0). */
typedef struct {
    int32_t nbins;          /* > 0: record the histogram */
    int64_t *hist;          /* [nprod_cap * nbins], nullable */
    int64_t *ntasks;        /* [nprod_cap], nullable */
    int32_t *ikj;           /* [3 * ikj_cap], nullable */
    int64_t ikj_cap;
    int64_t nprod_cap;
    int64_t nprod;          /* out (zero it before attaching) */
    int64_t ikj_count;      /* out */
    int64_t ikj_needed;     /* out */
} spamm_volume_sink;
/* sink == NULL detaches. */
spamm_status spamm_ctx_set_volume_sink(spamm_ctx ctx, spamm_volume_sink *sink);

/* -------------------------------------------------------- Newton-Schulz */
/* One dual step (north_star form): X = Z (x)_tau Y; t = (n - tr X)/n;
 * H = 1/2 (3I - X) (fused in the X epilogue, X is never stored);
 * Y' = Y (x)_tau_s H; Z' = H (x)_tau Z.  H_out nullable (else freed). */
spamm_status spamm_ns_step(spamm_ctx ctx, spamm_mat Y, spamm_mat Z, double tau, double tau_s,
                           spamm_mat *Y_next, spamm_mat *Z_next, spamm_mat *H_out,
                           double *t_k /* host, nullable */, spamm_stats stats[3] /* nullable */);
/* spamm_ns_step with a choice of NS map (see spamm_ns_opts.map):
 *   map 1: x~ = (1 - 2 eps) X + eps I, H = sqrt(alpha)/2 (3I - alpha x~), with
 *   alpha(t) = 1 + 1.85/(1 + e^{-50(t-.35)}), eps(t) = .1/(1 + e^{-75(t-.30)}) evaluated
 *   on the device at t = t_k.  X is stored by the GEMM epilogue and mapped
 *   in place by a second pass (the coefficients need the complete trace).
 *   alpha_eps: host [2] (alpha, eps) used, nullable.  Errors as spamm_ns_step, plus
 *   EINVAL for map not in {0, 1}. */
spamm_status spamm_ns_step_map(spamm_ctx ctx, spamm_mat Y, spamm_mat Z, double tau, double tau_s,
                               int32_t map, spamm_mat *Y_next, spamm_mat *Z_next, spamm_mat *H_out,
                               double *t_k, spamm_stats stats[3], double *alpha_eps);
/* Single-channel square-root iteration (Eq. single; the sensitive product
 * rightmost), one step from (Z_k, H_k = h[X_k]) with s' = s/c:
 *   Z_{k+1} = Z_k (x)_tau H_k,  W = s' (x)_tau_s Z_{k+1},  H_{k+1} = h[Z_{k+1}^T (x)_tau W],
 * t_next = (n - tr X_{k+1})/n; map as in spamm_ns_step_map.  W_out nullable.
 * stats[3] = (Z H, s' Z, Z^T W).  Not available on a row-partitioned context. */
spamm_status spamm_ns_step_single(spamm_ctx ctx, spamm_mat S1, spamm_mat Z, spamm_mat H, double tau,
                                  double tau_s, int32_t map, spamm_mat *Z_next, spamm_mat *H_next,
                                  spamm_mat *W_out, double *t_next, spamm_stats stats[3],
                                  double *alpha_eps);
/* Full single-channel run: c (power iteration or opts->scale), Z_0 = I, X_0 = s/c,
 * iters steps (opts: tau_s, map, t_stop, histories as spamm_ns_sqrt; mu must be 0),
 * outputs Z * c^{-1/2} -> s^{-1/2} and Y = W c^{1/2} -> s^{1/2}. */
spamm_status spamm_ns_sqrt_single(spamm_ctx ctx, spamm_mat s, double tau, int32_t iters, spamm_mat *Y,
                                  spamm_mat *Z, const spamm_ns_opts *opts);
/* Regularised product representation of the inverse factor (Eq. product_rep,
 * P:748-776; reading L21): slices of shifted,
 * preconditioned residuals, each "effective by one order":
 *   c = ||s||_2 (power iteration, or scale > 0), S_i = s/c + mu_i I,
 *   R_0 = S_0, R_i = F^T (x)_tau1 (S_i (x)_tau1 F) for i >= 1,
 *   Z_i = R_i^{-1/2} by the dual iteration (tau = tau_s = tau0, up to iters steps,
 *   t_stop as in spamm_ns_opts), F = Z_0, F <- F (x)_tau1 Z_i;
 *   *G = F / sqrt(c), so that G^T (s + c mu_{m} I) G ~ I.
 * mu: HOST [nslices], relative shifts, decreasing.  c_out, slice_iters ([nslices]) nullable.
 * Single device only (EINVAL on a row-partitioned context). */
spamm_status spamm_regularized_factor(spamm_ctx ctx, spamm_mat s, double tau0, double tau1, const double *mu,
                                      int32_t nslices, int32_t iters, double t_stop, double scale, spamm_mat *G,
                                      double *c_out, int32_t *slice_iters);
/* Scale estimate c ~ ||s||_2 ("easily obtained largest eigenvalue"; DESIGN.md
 * reading L12): K power steps v <- w/||w||, w = s v, from v_0 = 1/sqrt(n) * ones, then the
 * Rayleigh quotient c = v^T s v; every sum in a fixed order (deterministic).  s is read
 * as stored: when it is bitwise symmetric (checked on the device once per call) only its
 * blocks on and above the block diagonal are streamed (half the HBM traffic, same
 * result up to summation order); otherwise all of it.  *c: host.  Synchronises. */
spamm_status spamm_power_scale(spamm_ctx ctx, spamm_mat s, int32_t K, double *c);
/* Y0 = s/c (mu = 0) or (s/c + mu I)/(1+mu). */
spamm_status spamm_ns_y0(spamm_ctx ctx, spamm_mat s, double c, double mu, spamm_mat *Y0);
/* Identity quadtree (diagonal blocks = I). */
spamm_status spamm_identity(spamm_ctx ctx, int64_t n, int32_t b, spamm_mat *I);
/* Full run: setup (c, Y0 = s/c, Z0 = I), iters dual steps, unscale
 * (Y * sqrt(c(1+mu)), Z / sqrt(c(1+mu))).  On ENOTFINITE, Y/Z hold the last finite
 * iterates (unscaled) and t_history is filled up to the failing step. */
spamm_status spamm_ns_sqrt(spamm_ctx ctx, spamm_mat s, double tau, int32_t iters, spamm_mat *Y,
                           spamm_mat *Z, const spamm_ns_opts *opts);
/* m * alpha (divide = 0) or m / alpha (divide = 1), new matrix, same pattern. */
spamm_status spamm_scale(spamm_ctx ctx, spamm_mat m, double alpha, int32_t divide,
                         spamm_mat *out);

/* Write all stored blocks: bi/bj [cap] (int32), blocks [cap*b*b] (host or device);
 * *n = number of stored blocks (pool order).  Pass cap = 0 to query *n. */
spamm_status spamm_export_blocks(spamm_ctx ctx, spamm_mat m, int32_t *bi, int32_t *bj,
                                 double *blocks, int64_t cap, int64_t *n);
/* Asynchronous spamm_export_blocks to HOST buffers (pinned for real overlap): the
 * row-major staging runs on the context stream into a library-owned device slot
 * (SPAMM_XSLOTS = 4 of them, reused round-robin, each grown on demand), the
 * device->host copy on the context's own copy stream, so it overlaps whatever the
 * context stream runs next.  m may be freed right after the call.  The host buffers
 * are complete after spamm_copies_wait (host) or, in stream order, after
 * spamm_copies_join (the context stream waits for every export issued so far).
 * Errors: EINVAL (device output pointers, NULL), ENOMEM (staging). */
spamm_status spamm_export_blocks_async(spamm_ctx ctx, spamm_mat m, int32_t *bi, int32_t *bj,
                                       double *blocks, int64_t cap, int64_t *n);
spamm_status spamm_copies_join(spamm_ctx ctx);
spamm_status spamm_copies_wait(spamm_ctx ctx);

/* Asynchronous upload of a block-list input from HOST memory (pinned for overlap),
 * the prefetch half of spamm_build_tree_blocks: the host->device copy is issued at
 * once on the library's upload stream, into one of SPAMM_ISLOTS = 2 context-owned
 * staging slots (round-robin; a slot is refilled only after the build that read it),
 * with NO ordering against the context stream, so it overlaps whatever the context is
 * computing.  spamm_build_tree_staged(ctx, n, staged, &m) then builds the quadtree
 * on the context stream once the copy has landed (same result as
 * spamm_build_tree_blocks on the same arrays) and consumes the handle; the host
 * arrays must stay unchanged until then.  At most SPAMM_ISLOTS uploads may be
 * outstanding (an older handle is rejected with EINVAL).  spamm_staged_free drops an
 * unused handle.  Errors: EINVAL (device pointers, b), ENOMEM (staging). */
typedef struct spamm_staged_s *spamm_staged;
spamm_status spamm_stage_blocks(spamm_ctx ctx, int64_t nblocks, int32_t b, const int32_t *bi,
                                const int32_t *bj, const double *blocks, spamm_staged *out);
/* the same for a dense n x n row-major HOST input with leading dimension ld (the
 * prefetch half of spamm_build_tree) */
spamm_status spamm_stage_dense(spamm_ctx ctx, const double *dense, int64_t n, int64_t ld, spamm_staged *out);
/* b must equal the block-list upload's; for a dense upload n must equal its n */
spamm_status spamm_build_tree_staged(spamm_ctx ctx, int64_t n, int32_t b, spamm_staged staged, spamm_mat *out);
void spamm_staged_free(spamm_staged staged);

/* ------------------------------------------------- measurement utilities */
/* Device-side phase timing with CUDA events on the context stream (bench.py
 * uses it for the roofline of the dominant kernel).  Phases: */
enum { SPAMM_PH_GEMM = 0, SPAMM_PH_CULL = 1, SPAMM_PH_SETUP = 2, SPAMM_PH_LOOP = 3,
       SPAMM_PH_OTHER = 4, SPAMM_NPHASE = 5 };
typedef struct {
    double ms[SPAMM_NPHASE];        /* summed event time per phase            */
    int64_t count[SPAMM_NPHASE];    /* number of timed intervals per phase    */
    double gemm_flops;              /* sum of 2 b^3 |S| over timed GEMMs      */
    int64_t gemm_tasks;
    double gemm_operand_bytes;      /* 2 * 8 b^2 |S| + 8 b^2 segments (algorithmic) */
} spamm_profile_t;
spamm_status spamm_profile_enable(spamm_ctx ctx, int32_t enable);  /* resets the counters */
spamm_status spamm_profile_read(spamm_ctx ctx, spamm_profile_t *out); /* syncs */
/* FP64 DMMA issue-rate microbenchmark: TFLOP/s of back-to-back independent
 * mma.sync.m8n8k4.f64 on all SMs for `iters` per warp (syncs). */
spamm_status spamm_peak_dmma(spamm_ctx ctx, int64_t iters, double *tflops, double *ms);

#ifdef __cplusplus
}
#endif
#endif /* SPAMM_B200_H */
