// common.cuh — internal types and helpers of libspamm_b200 (sm_100a only).
//
// HBM layout of one quadtree matrix:
//   norm2 : fp64 squared-Frobenius pyramid, level l (0 = root .. L = leaves)
//           at offset pyr_off(l), 4^l entries in Morton order, so the four
//           children of node m are the 32-byte sector 4m..4m+3 of level l+1
//           (P:125-129 stored squared, reading L5).
//   slot  : int32 [nb*nb] Morton order -> pool slot, -1 = absent block.
//   pool  : fp64 [cap][b*b], each leaf block row-major with its 16-byte chunks
//           XOR-swizzled inside each row (pool_at below), 256-B aligned.  A
//           linear TMA bulk copy of a block therefore lands in shared memory
//           already in the bank-conflict-free layout the DMMA fragment loads want.
//   coord : int32 [cap] Morton code of the block in each pool slot.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/spamm.h"

#define SPAMM_MAX_L 15
#define SPAMM_MAX_WORLD 64

// Row partition of the leaf block rows over the ranks of a communicator
// (SURVEY.md §8(e)): rank p owns block rows [rs[p], rs[p+1]).
struct Parts {
    int world;
    int rs[SPAMM_MAX_WORLD + 1];
};

// Transport of the row-partitioned path (comm.cu): NCCL over NVLink, or an
// in-process group of host threads (one context per thread) used to run G
// ranks on one device for the determinism tests.  Both are stream-ordered on
// the calling context's stream.
struct spamm_comm_s {
    int rank = 0, world = 1;
    virtual ~spamm_comm_s() {}
    // recv[p*bytes .. (p+1)*bytes) <- rank p's send (all ranks, rank order)
    virtual spamm_status allgather(spamm_ctx ctx, const void *send, void *recv, size_t bytes) = 0;
    // rank p receives scnt[p] bytes from send + soff[p]; from rank p, rcnt[p]
    // bytes arrive at recv + roff[p] (offsets / counts in bytes, host arrays)
    virtual spamm_status alltoallv(spamm_ctx ctx, const void *send, const size_t *soff,
                                   const size_t *scnt, void *recv, const size_t *roff,
                                   const size_t *rcnt) = 0;
    virtual const char *kind() const = 0;
    // Peer memory: a rank's kernels may read another rank's device
    // memory directly (same process; the same device or peer access over NVLink).
    // peer_share publishes n device pointers, returns every rank's (rank-major in all),
    // and makes the calling stream wait for the work every rank queued before the call
    // (so the memory behind the pointers is complete); *ok = 0 when some pair of ranks
    // cannot access each other's memory.  peer_barrier: the calling stream waits for the
    // work every rank queued before the call (readers are done before an owner reuses
    // or frees what it shared).
    virtual bool peer_capable() const { return false; }
    virtual spamm_status peer_share(spamm_ctx, const void *const *, int, const void **, int *ok)
    {
        *ok = 0;
        return SPAMM_OK;
    }
    virtual spamm_status peer_barrier(spamm_ctx) { return SPAMM_OK; }
};

struct spamm_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    spamm_allocator alloc{};
    bool has_alloc = false;
    cudaMemPool_t pool = nullptr;   // the context's stream-ordered pool (no allocator given)
    std::string err;
    int64_t launches = 0;
    int sm_count = 148;
    // last product's leaf tasks (for spamm_export_tasks)
    struct Cull *last = nullptr;
    // cull workspaces owned by the context (grown on demand), one per product role
    struct Cull *cw[3] = {nullptr, nullptr, nullptr};
    double *dscratch = nullptr;   // small device scratch (norms, trace, t)
    int64_t *iscratch = nullptr;  // small device scratch (counters)
    double *hpinned = nullptr;    // pinned host scratch
    void *prof = nullptr;         // prof.cu state
    // row-partitioned execution (dist.cu); comm == nullptr => single device
    spamm_comm comm = nullptr;
    std::vector<int> row_start;   // [world+1] block rows; empty => equal split per nb
    struct Dist *dist = nullptr;  // exchange workspaces
    cudaStream_t comm_stream = nullptr;   // halo exchange overlapped with the local GEMM
    void *zc = nullptr;            // mapped pinned host buffer for small device->host reads
    void *zc_dev = nullptr;        // its device alias
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    // matrices allocated from this context and not yet freed; spamm_ctx_destroy with
    // live matrices defers the teardown to the last spamm_mat_free (their memory
    // comes from the context's pool / allocator)
    spamm_volume_sink *vsink = nullptr;   // per-product recorder (f4), nullable
    struct NsGraph *nsg = nullptr;        // cached graph-replayed NS step (spamm.cu)
    void *xs = nullptr;                   // asynchronous export: copy stream + staging (prof.cu)
    bool capturing = false;               // inside a CUDA graph capture (no prof events)
    int gemm_grid_cap = 0;                // > 0: at most this many leaf-GEMM CTAs (overlap window)
    std::atomic<int64_t> live_mats{0};
    std::atomic<bool> destroy_pending{false};
};
// tear down a context whose matrices are all freed (spamm.cu)
void ctx_teardown(spamm_ctx ctx);

struct spamm_mat_s {
    spamm_ctx ctx = nullptr;
    int64_t n = 0;
    int b = 0, nb = 0, L = 0;
    double *norm2 = nullptr;   // pyramid
    int32_t *slot = nullptr;   // nb*nb Morton
    double *pool = nullptr;    // cap * b*b
    int32_t *coord = nullptr;  // cap
    int64_t nblk = 0, cap = 0;
    // row partition: this rank stores block rows [r0, r1); the norm pyramid and
    // the leaf-norm level are complete (replicated) on every rank.
    int r0 = 0, r1 = 0;
    bool dist = false;
    Parts parts{};
};

// ------------------------------------------------------------------ memory
void *dev_alloc(spamm_ctx ctx, size_t bytes);
void dev_free(spamm_ctx ctx, void *p, size_t bytes);

template <typename T>
static inline T *dalloc(spamm_ctx ctx, int64_t count)
{
    return (T *)dev_alloc(ctx, sizeof(T) * (size_t)(count > 0 ? count : 1));
}

// Pyramid level offsets, padded so every level starts on a 32-byte sector:
// off(0) = 0 (root, padded to 4 entries), off(l) = (4^l + 8)/3 for l >= 1.
__host__ __device__ static inline int64_t pyr_off(int l)
{
    return l == 0 ? 0 : ((int64_t(1) << (2 * l)) + 8) / 3;
}
__host__ __device__ static inline int64_t pyr_size(int L)
{
    return L == 0 ? 4 : pyr_off(L) + (int64_t(1) << (2 * L));
}

// ------------------------------------------------------------ debug asserts
// Built with -DSPAMM_DEBUG (paper_1508_05856_b200/_build.py build_debug -> the
// libspamm_b200_debug.so that SPAMM_LIB can select): device-side bounds checks on
// every index that addresses a pool, a task list or a slot map; a failure prints the
// condition and traps (the launch fails with an error the host reports).  Compiled out
// of the product library.
#ifdef SPAMM_DEBUG
#include <cstdio>
#define SPAMM_ASSERT(c)                                                                             \
    do {                                                                                          \
        if (!(c)) {                                                                               \
            printf("SPAMM_ASSERT(%s) failed at %s:%d block %d thread %d\n", #c, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                            \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define SPAMM_ASSERT(c) \
    do {                \
    } while (0)
#endif

// ------------------------------------------------------------------ Morton
__host__ __device__ static inline uint32_t spread_bits(uint32_t x)
{
    x &= 0xFFFF;
    x = (x | (x << 8)) & 0x00FF00FF;
    x = (x | (x << 4)) & 0x0F0F0F0F;
    x = (x | (x << 2)) & 0x33333333;
    x = (x | (x << 1)) & 0x55555555;
    return x;
}
__host__ __device__ static inline uint32_t compact_bits(uint32_t x)
{
    x &= 0x55555555;
    x = (x | (x >> 1)) & 0x33333333;
    x = (x | (x >> 2)) & 0x0F0F0F0F;
    x = (x | (x >> 4)) & 0x00FF00FF;
    x = (x | (x >> 8)) & 0x0000FFFF;
    return x;
}
// row index i in the odd bits, column j in the even bits: children of m are 4m + (di<<1|dj)
__host__ __device__ static inline uint32_t morton(uint32_t i, uint32_t j)
{
    return (spread_bits(i) << 1) | spread_bits(j);
}
__host__ __device__ static inline uint32_t morton_i(uint32_t m) { return compact_bits(m >> 1); }
__host__ __device__ static inline uint32_t morton_j(uint32_t m) { return compact_bits(m); }

// ------------------------------------------------------------------ pool swizzle
// Element (r, c) of a b x b block lives at pool_at(r, c): the 16-byte chunk c/2 of
// row r is stored at chunk (c/2) ^ swz(r), swz(r) = ((r>>2)&3)<<1 | (r&1) in [0,8).
// Both DMMA fragment patterns are then conflict-free: A (lane (g,t) reads
// A[g][4t..4t+3], two LDS.128) and B (lane (g,t) reads B[4t+s][g], LDS.64; rows
// s, s+4, s+8, s+12 of a half-warp hit four different bank groups).
__host__ __device__ static inline int swz(int r) { return (((r >> 2) & 3) << 1) | (r & 1); }
__host__ __device__ static inline int pool_at(int r, int c, int b)
{
    return r * b + ((((c >> 1) ^ swz(r)) << 1) | (c & 1));
}
// inverse: physical offset e -> logical column of that element
__host__ __device__ static inline int pool_col(int e, int b)
{
    int r = e / b, q = e % b;
    return ((((q >> 1) ^ swz(r)) << 1) | (q & 1));
}

// Programmatic dependent launch, for chains of small dependent kernels on one stream
// (the cull's levels, the power iteration): each kernel lets its successor launch at
// once (griddepcontrol.launch_dependents) and each successor waits for its
// predecessor's completion and memory (griddepcontrol.wait) before touching anything,
// so the next launch's latency overlaps this kernel's tail.  Without the launch
// attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// SPAMM_PDL=0 turns the attribute off (plain stream-ordered launches)
static inline bool pdl_enabled()
{
    static const bool on = [] {
        const char *e = getenv("SPAMM_PDL");
        return !(e && *e == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// with PDL on a single device; a plain launch when the context has a communicator
// (row partition: the predecessor on the stream may be a collective or a copy)
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(spamm_ctx ctx, void (*k)(KArgs...), int grid, int block, size_t smem, Args... args)
{
    if (ctx->comm == nullptr) return launch_pdl(k, grid, block, smem, ctx->stream, args...);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------ small device->host reads
// Counts and scalars are read back through a kernel that stores into mapped pinned
// host memory, not cudaMemcpy: a small D2H copy queues behind any large transfer on
// the copy engine (e.g. a caller streaming the previous result to the host), while a
// kernel's stores go straight over the bus.  One launch + one stream sync per call.
#define SPAMM_ZC_BYTES 65536
struct FetchItem {
    const void *src;   // device
    void *dst;         // host
    uint32_t bytes;    // multiple of 4
};
spamm_status fetch(spamm_ctx ctx, const FetchItem *items, int n);
static inline spamm_status fetch1(spamm_ctx ctx, const void *src, void *dst, uint32_t bytes)
{
    FetchItem it{src, dst, bytes};
    return fetch(ctx, &it, 1);
}

// ------------------------------------------------------------------ errors
spamm_status set_err(spamm_ctx ctx, spamm_status st, const char *fmt, ...);
spamm_status check_cuda(spamm_ctx ctx, cudaError_t e, const char *what);
#define CK(call)                                                              \
    do {                                                                      \
        cudaError_t _e = (call);                                              \
        if (_e != cudaSuccess) return check_cuda(ctx, _e, #call);             \
    } while (0)
#define SPAMM_STR2(x) #x
#define SPAMM_STR(x) SPAMM_STR2(x)
#define CKL(ctx)                                                              \
    do {                                                                      \
        (ctx)->launches++;                                                    \
        cudaError_t _e = cudaGetLastError();                                  \
        if (_e != cudaSuccess)                                                \
            return check_cuda(ctx, _e, "kernel launch at " __FILE__ ":" SPAMM_STR(__LINE__)); \
    } while (0)
#define ST(call)                                                              \
    do {                                                                      \
        spamm_status _s = (call);                                             \
        if (_s != SPAMM_OK) return _s;                                        \
    } while (0)

static inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// SMs left to the halo exchange while the local-segment GEMM runs (row partition,
// world > 1); NCCL communicators are created with maxCTAs = this (SPAMM_EXCHANGE_CTAS,
// default 8)
static inline int exchange_ctas()
{
    static const int v = [] {
        const char *e = getenv("SPAMM_EXCHANGE_CTAS");
        const int x = e && *e ? atoi(e) : 8;
        return x < 1 ? 1 : x > 64 ? 64 : x;
    }();
    return v;
}

// Per-device, thread-safe one-time kernel configuration (function attributes are
// per device; contexts may be driven from several host threads).  f() is
// idempotent, so two threads racing on the first call both running it is harmless.
template <typename F>
static inline cudaError_t once_per_device(std::atomic<uint64_t> &done, int device, F &&f)
{
    const uint64_t bit = 1ull << (device & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    cudaError_t e = f();
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    return e;
}

// ------------------------------------------------------------ internal API
// tree.cu
spamm_status mat_new(spamm_ctx ctx, int64_t n, int b, int64_t cap, spamm_mat *out);
spamm_status mat_reset_pattern(spamm_ctx ctx, spamm_mat m);     // slot=-1, leaf norms=0
spamm_status pyramid_build(spamm_ctx ctx, spamm_mat m);           // levels L-1..0 from leaves
spamm_status pyramid_build_pair(spamm_ctx ctx, spamm_mat m, spamm_mat m2);   // two, one launch per pass
spamm_status mat_map(spamm_ctx ctx, spamm_mat src, int op, double c, double mu, spamm_mat *out);
int is_device_ptr(const void *p);

// dist.cu — the row-partitioned path
spamm_status mat_parts(spamm_ctx ctx, int nb, Parts *p);          // partition of nb block rows
// leaf norms of the local rows -> replicated on all ranks, then the pyramid
spamm_status norms_finish(spamm_ctx ctx, spamm_mat m);
// gather rows of a vector laid out as nb rows x width (row-major) across ranks
spamm_status gather_rows(spamm_ctx ctx, const Parts &p, double *vec, int width);
// fetch the remote right-operand blocks the local tasks of cw use; patches
// cw->tB (remote => -(h+1), h = halo slot) and returns the halo pool
spamm_status halo_exchange(spamm_ctx ctx, struct Cull *cw, spamm_mat B, double **halo, int64_t *nhalo);
// peer memory (§8(e) v3): when every rank can read every other's memory, resolve the
// remote tasks' B slots in the owners' slot maps and point the GEMM at the owners'
// pools (cw->peer_*); *used = false => use halo_exchange.  The caller runs
// comm->peer_barrier after the GEMM (owners keep their B until every reader is done).
spamm_status peer_patch(spamm_ctx ctx, struct Cull *cw, spamm_mat B, bool *used);
// stable split of the segments into all-local (every task's B block is row-local)
// then remote-using ones: order[nsegs] (device, caller frees), *nlocal (host)
spamm_status seg_split(spamm_ctx ctx, struct Cull *cw, int32_t **order, int64_t *nlocal);
void dist_free(spamm_ctx ctx);

// cull.cu — the level-by-level two-sided norm query (Eq. newspamm)
enum { CNT_OVERFLOW = 16, CNT_NSEG = 17, CNT_TICKET = 20, CNT_GEMM_TICKET = 48 };  // counters[] layout; [0..15] = level counts
struct Cull {
    int64_t cap = 0;              // task capacity of every level
    int64_t cap_segs = 0;         // segment capacity
    int4 *rec[2] = {nullptr, nullptr};  // ping-pong level records {code(I,J), K, gstart, gend}
    int4 *pre = nullptr;          // per-task exclusive scan of child counts per quadrant [cap+1]
    uint8_t *mask = nullptr;      // per-task 8-bit child mask, bit (2q + dk)
    int32_t *tA = nullptr, *tB = nullptr, *tK = nullptr;  // final tasks: A slot, B slot, k
    int32_t *seg_code = nullptr, *seg_start = nullptr, *seg_len = nullptr;
    int64_t tiles = 0;            // tiles per scan
    int32_t *tile_flag = nullptr; // [(SPAMM_MAX_L + 2) * tiles]
    int4 *tile_agg = nullptr, *tile_pre = nullptr;  // [tiles]
    int32_t *counters = nullptr;  // [64] device
    int32_t *hcnt = nullptr;      // [64] pinned host mirror
    int final_buf = 0;            // rec[] index holding the leaf-level records
    int L = 0, l0 = 0, b = 0;
    int64_t ntasks = 0, nsegs = 0;  // host copies after cull_sync
    int64_t hint = 0;             // capacity hint for the next use
    // level sizes of the previous accepted query on this workspace (grid sizing of the
    // next one: consecutive NS products of one role have similar levels; the kernels
    // loop over their work, so any grid is correct)
    int prevL = -1;
    int32_t prev[SPAMM_MAX_L + 2] = {};
    double alpha = 1.0;           // EPI_STORE output scale of the next GEMM (fused unscale)
    int64_t gen = 0;              // bumped by every (re)allocation (captured graphs check it)
    bool counts_only = false;     // a counting query (its tasks never reach a GEMM)
    // peer memory (dist.cu peer_patch): remote right-operand tiles are read in place from
    // the owners' pools; tB = -(slot * peer_world + owner) - 1 for those tasks
    int peer_world = 0;
    const double *peer_pool[SPAMM_MAX_WORLD] = {};
    spamm_stats stats{};
};
// Enqueue the query, synchronise once to read the counts, and grow + re-run
// on capacity overflow.
spamm_status cull_run(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int r0, int r1,
                      int transA = 0);
spamm_status cull_start(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int r0, int r1,
                        int transA = 0);
// arrays the query's first kernel clears (device-driven steps): slot maps -> -1,
// pyramids -> 0 of up to 3 output matrices, and z[0..nz) -> 0
struct CullClear {
    int32_t *slot[3];
    double *n2[3];
    int64_t nslot, nn2;
    double *z;
    int64_t nz;
};
spamm_status cull_clear_enqueue(spamm_ctx ctx, const CullClear &clr);
// enqueue only (fixed workspace, capacity-sized grids): for CUDA graph capture
spamm_status cull_enqueue_fixed(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau,
                                const CullClear *clear = nullptr);
// (re)allocate a workspace for at least cap tasks per level and cap_segs segments
spamm_status cull_reserve(spamm_ctx ctx, Cull *cw, int64_t cap, int64_t cap_segs);
spamm_status cull_complete(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int r0, int r1,
                           int transA = 0);
void cull_free(spamm_ctx ctx, Cull *cw);
spamm_status cull_export(spamm_ctx ctx, Cull *cw, int32_t *ikj_host, int64_t cap, int64_t *n);
// append this product's record to ctx->vsink (no-op without a sink)
spamm_status volume_record(spamm_ctx ctx, Cull *cw);

// gemm.cu — FP64 DMMA leaf GEMM with fused epilogues
enum { EPI_STORE = 0, EPI_NS_H = 1, EPI_NS_X = 2 };
// seg_order (nullable) / nseg (< 0 => all cw->nsegs) select the segments of this launch;
// ticket = which of the GEMM ticket counters (zeroed by the cull) the launch uses
// device_count: the launch reads the segment count from cw->counters (device-driven
// steps, CUDA graph capture) and runs a full persistent grid
spamm_status gemm_run(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, const double *b_halo,
                      spamm_mat C, int epi, double *trace_part, const int32_t *seg_order = nullptr,
                      int64_t nseg = -1, int ticket = 0, int transA = 0, bool device_count = false);
spamm_status gemm_run_pair(spamm_ctx ctx, struct Cull *c1, spamm_mat A1, spamm_mat B1, spamm_mat C1,
                           struct Cull *c2, spamm_mat A2, spamm_mat B2, spamm_mat C2);
// diag_fixup with the base slot read from the device (the X cull's segment count) and
// caller-provided scratch (newslot [nb]); no allocation, no host round trip
spamm_status diag_fixup_dev(spamm_ctx ctx, spamm_mat H, const int32_t *nseg_dev, double value, int32_t *newslot,
                            int64_t *dcount, const double *trace_part = nullptr, double *t_out = nullptr);
spamm_status diag_fixup(spamm_ctx ctx, spamm_mat H, int64_t nseg, double value);
// as diag_fixup without the host round trip: the count of appended blocks lands in
// *dcount (device); the caller fetches it and sets H->nblk = nseg + count
// trace_part (nullable): the fill launch also forms t_k = (n - sum trace_part)/n -> *t_out
// (trace_finish's arithmetic; single device)
spamm_status diag_fixup_async(spamm_ctx ctx, spamm_mat H, int64_t nseg, double value, int64_t *dcount,
                              const double *trace_part = nullptr, double *t_out = nullptr);
// out[0..n) = the segments of `in` (nullable => 0..n-1), longest first (a schedule only)
spamm_status lpt_order(spamm_ctx ctx, const int32_t *seg_len, const int32_t *in, int64_t n, int32_t *out);
// scaled / stabilised NS map in place over X: coef <- {alpha, eps, sqrt(alpha)/2}(t)
spamm_status ns_scaled_map(spamm_ctx ctx, spamm_mat X, const double *t, double *coef);
// append value*I blocks for absent diagonal positions at slots base..; *added = count (syncs)
spamm_status diag_append(spamm_ctx ctx, spamm_mat m, int64_t base, double value, int64_t *added);
spamm_status trace_finish(spamm_ctx ctx, const double *trace_part, int nb, int64_t n,
                          double *t_out);

// prof.cu — phase timing (no-ops unless spamm_profile_enable)
int prof_begin(spamm_ctx ctx, int phase);
void prof_end(spamm_ctx ctx, int idx);
void prof_gemm_work(spamm_ctx ctx, int64_t tasks, int64_t segs, int b);
void prof_destroy(spamm_ctx ctx);
#define SPAMM_XSLOTS 4
#define SPAMM_ISLOTS 2
void xstate_free(spamm_ctx ctx);   // the asynchronous host-I/O state (hostio.cu; copies drained first)

// power.cu
spamm_status power_scale(spamm_ctx ctx, spamm_mat s, int K, double *c_host);
