// spamm.cu — the C ABI entry points: context, SpAMM product, Newton-Schulz.
//
//   spamm_multiply : C = A (x)_tau B   (Eq. newspamm)
//       cull (cull.cu) -> one stream sync for the counts -> DMMA leaf GEMM with
//       the store epilogue (gemm.cu) -> norm pyramid of C (tree.cu)
//   spamm_ns_step  : X = Z (x)_tau Y (epilogue writes H = 1/2(3I - X) and tr X
//       partials), diagonal fix-up, t_k; Y' = Y (x)_tau_s H; Z' = H (x)_tau Z
//       (Eq. cannonical P:383-389 in the north_star form, reading L8)
//   spamm_ns_sqrt  : setup (c, Y0 = s/c, Z0 = I) + iters steps + unscale.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

static void ns_graph_free(spamm_ctx ctx);

extern "C" spamm_status spamm_ctx_create(int device, void *cuda_stream, const spamm_allocator *allocator,
                                         spamm_ctx *out)
{
    if (!out) return SPAMM_EINVAL;
    *out = nullptr;
    spamm_ctx ctx = new spamm_ctx_s();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete ctx;
        return SPAMM_ECUDA;
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (major != 10 || minor != 0) {
        delete ctx;
        return SPAMM_ECUDA;   // built for sm_100a only
    }
    if (cuda_stream) ctx->stream = (cudaStream_t)cuda_stream;
    else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete ctx;
            return SPAMM_ECUDA;
        }
        ctx->own_stream = true;
    }
    if (allocator && allocator->alloc && allocator->free) {
        ctx->alloc = *allocator;
        ctx->has_alloc = true;
    } else {
        // stream-ordered allocator: keep freed memory in the pool across synchronisations
        // (the default release threshold of 0 returns it to the driver at every sync, and
        // the next cudaMallocAsync pays for a fresh mapping: C3 ran 8x slower that way)
        // A pool of the context's own (not the device's default pool, which other users
        // of the process may trim or share).
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        if (cudaMemPoolCreate(&ctx->pool, &props) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr);
        } else {
            ctx->pool = nullptr;
        }
        cudaGetLastError();
    }
    ctx->dscratch = dalloc<double>(ctx, 64);
    ctx->iscratch = dalloc<int64_t>(ctx, 64);
    if (!ctx->dscratch || !ctx->iscratch) {
        delete ctx;
        return SPAMM_ENOMEM;
    }
    for (int i = 0; i < 3; i++) ctx->cw[i] = new Cull();
    *out = ctx;
    return SPAMM_OK;
}

extern "C" void spamm_ctx_destroy(spamm_ctx ctx)
{
    if (!ctx) return;
    // matrices still alive: they own memory of this context (its pool / allocator) and
    // point back at it, so the teardown waits for the last spamm_mat_free
    ns_graph_free(ctx);   // its buffers are matrices of this context
    ctx->destroy_pending.store(true);
    if (ctx->live_mats.load() > 0) return;
    ctx_teardown(ctx);
}

void ctx_teardown(spamm_ctx ctx)
{
    cudaStreamSynchronize(ctx->stream);
    xstate_free(ctx);
    dist_free(ctx);
    for (int i = 0; i < 3; i++) {
        if (!ctx->cw[i]) continue;
        cull_free(ctx, ctx->cw[i]);
        dev_free(ctx, ctx->cw[i]->counters, sizeof(int32_t) * 64);
        if (ctx->cw[i]->hcnt) cudaFreeHost(ctx->cw[i]->hcnt);
        delete ctx->cw[i];
    }
    if (ctx->zc) cudaFreeHost(ctx->zc);
    dev_free(ctx, ctx->dscratch, sizeof(double) * 64);
    dev_free(ctx, ctx->iscratch, sizeof(int64_t) * 64);
    cudaStreamSynchronize(ctx->stream);
    prof_destroy(ctx);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

extern "C" const char *spamm_last_error(spamm_ctx ctx) { return ctx ? ctx->err.c_str() : "no context"; }

extern "C" int64_t spamm_kernel_launches(spamm_ctx ctx) { return ctx ? ctx->launches : 0; }

static spamm_status check_pair(spamm_ctx ctx, spamm_mat A, spamm_mat B, double tau)
{
    if (!ctx || !A || !B) return set_err(ctx, SPAMM_EINVAL, "NULL argument");
    if (A->n != B->n || A->b != B->b)
        return set_err(ctx, SPAMM_ESHAPE, "shape mismatch: (n=%lld,b=%d) vs (n=%lld,b=%d)",
                       (long long)A->n, A->b, (long long)B->n, B->b);
    if (!(tau >= 0.0) || !std::isfinite(tau)) return set_err(ctx, SPAMM_EINVAL, "tau must be finite and >= 0");
    return SPAMM_OK;
}

// SPAMM_LPT=1 turns on a longest-first GEMM schedule (measured: -0.4 % GEMM time but
// +0.5 % step time on C3 from its three extra launches per product, and 4 % slower
// products at C5, where it breaks the Morton order's L2 reuse; off by default)
static int lpt_mode()
{
    static const int m = [] {   // initialised once, thread-safely (C++11)
        const char *e = getenv("SPAMM_LPT");
        return (e && *e == '1') ? 1 : 0;
    }();
    return m;
}

// ------------------------------------------------------------ self-check
// SPAMM_SELFCHECK=1 (debug): every product re-runs its cull and its leaf GEMM and
// compares the task lists / output blocks bitwise (both are deterministic by
// construction); mismatches are reported on stderr.
static int selfcheck_mode()
{
    static const int m = [] {   // initialised once, thread-safely (C++11)
        const char *e = getenv("SPAMM_SELFCHECK");
        return (e && *e == '1') ? 1 : 0;
    }();
    return m;
}

__global__ void k_cmp_words(const uint32_t *a, const uint32_t *b, int64_t n, unsigned long long *mism,
                            unsigned long long *first)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (a[i] != b[i]) {
            atomicAdd(mism, 1ull);
            atomicMin(first, (unsigned long long)i);
        }
}

static long long cmp_words(spamm_ctx ctx, const void *a, const void *b, int64_t bytes, long long *first_word)
{
    unsigned long long *d = dalloc<unsigned long long>(ctx, 2);
    unsigned long long h[2] = {0, ~0ull};
    cudaMemcpyAsync(d, h, sizeof h, cudaMemcpyHostToDevice, ctx->stream);
    k_cmp_words<<<296, 256, 0, ctx->stream>>>((const uint32_t *)a, (const uint32_t *)b, bytes / 4, d, d + 1);
    cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    dev_free(ctx, d, 16);
    *first_word = (long long)h[1];
    return (long long)h[0];
}

static void *snapshot(spamm_ctx ctx, const void *src, int64_t bytes)
{
    void *p = dev_alloc(ctx, bytes > 0 ? bytes : 1);
    if (bytes > 0) cudaMemcpyAsync(p, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
    return p;
}

static std::atomic<int64_t> g_product_id{0};   // SELFCHECK log label (ranks may be threads)

static void selfcheck_cull(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int transA)
{
    const int64_t nt = cw->ntasks, ns = cw->nsegs;
    void *tA = snapshot(ctx, cw->tA, 4 * nt), *tB = snapshot(ctx, cw->tB, 4 * nt);
    void *sc = snapshot(ctx, cw->seg_code, 4 * ns), *ss = snapshot(ctx, cw->seg_start, 4 * ns),
         *sl = snapshot(ctx, cw->seg_len, 4 * ns);
    cull_run(ctx, cw, A, B, tau, A->r0, A->r1, transA);
    long long f[5], m[5];
    m[0] = cw->ntasks == nt && cw->nsegs == ns ? 0 : -1;
    if (!m[0]) {
        m[0] = cmp_words(ctx, tA, cw->tA, 4 * nt, &f[0]);
        m[1] = cmp_words(ctx, tB, cw->tB, 4 * nt, &f[1]);
        m[2] = cmp_words(ctx, sc, cw->seg_code, 4 * ns, &f[2]);
        m[3] = cmp_words(ctx, ss, cw->seg_start, 4 * ns, &f[3]);
        m[4] = cmp_words(ctx, sl, cw->seg_len, 4 * ns, &f[4]);
    } else {
        m[1] = m[2] = m[3] = m[4] = 0;
    }
    if (m[0] || m[1] || m[2] || m[3] || m[4])
        fprintf(stderr, "SELFCHECK cull mismatch product %lld: counts %lld/%lld vs %lld/%lld, tA %lld tB %lld code %lld start %lld len %lld\n",
                (long long)g_product_id.load(), (long long)nt, (long long)ns, (long long)cw->ntasks, (long long)cw->nsegs,
                m[0], m[1], m[2], m[3], m[4]);
    for (void *q : {tA, tB, sc, ss, sl}) dev_free(ctx, q, 1);
}

static void selfcheck_gemm(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, const double *halo, spamm_mat C,
                           int epi, int transA = 0)
{
    spamm_mat m2 = nullptr;
    if (mat_new(ctx, A->n, A->b, cw->nsegs + A->nb, &m2)) return;
    mat_reset_pattern(ctx, m2);
    double *tr = dalloc<double>(ctx, A->nb);
    cudaMemsetAsync(tr, 0, sizeof(double) * A->nb, ctx->stream);
    cudaMemsetAsync(cw->counters + CNT_GEMM_TICKET, 0, sizeof(int32_t), ctx->stream);
    gemm_run(ctx, cw, A, B, halo, m2, epi, tr, nullptr, -1, 0, transA);
    const int64_t b2 = (int64_t)A->b * A->b;
    long long f0, f1;
    long long m0 = cmp_words(ctx, C->pool, m2->pool, 8 * b2 * cw->nsegs, &f0);
    long long m1 = cmp_words(ctx, C->norm2 + pyr_off(C->L), m2->norm2 + pyr_off(C->L), 8 * (int64_t)A->nb * A->nb, &f1);
    if (m0 || m1)
        fprintf(stderr, "SELFCHECK gemm mismatch product %lld epi %d: pool words %lld (first block %lld), leaf n2 words %lld; tasks %lld segs %lld\n",
                (long long)g_product_id.load(), epi, m0, f0 / (2 * b2), m1, (long long)cw->ntasks, (long long)cw->nsegs);
    dev_free(ctx, tr, 8 * A->nb);
    spamm_mat_free(m2);
}

// Row partition, world > 1: GEMM over the all-local
// segments on the context stream || halo exchange on the communication stream,
// then the GEMM over the segments that use remote tiles.  Each segment is owned
// by one CTA and accumulated in ascending k, so the split changes no result.
// the context's second stream (+ events): the halo exchange (row partition) or the
// second of two concurrent culls (single device)
static spamm_status ensure_side_stream(spamm_ctx ctx)
{
    if (!ctx->comm_stream) {
        CK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
        for (auto &e : ctx->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return SPAMM_OK;
}

static spamm_status overlapped_gemm(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, spamm_mat m, int epi,
                                    double *trace_part)
{
    ST(ensure_side_stream(ctx));
    const cudaStream_t main_s = ctx->stream, comm_s = ctx->comm_stream;
    int32_t *order = nullptr;
    int64_t nloc = 0;
    ST(seg_split(ctx, cw, &order, &nloc));
    const int64_t nrem = cw->nsegs - nloc;
    // the exchange reads the cull's records / tB: comm stream after main
    CK(cudaEventRecord(ctx->ev[0], main_s));
    CK(cudaStreamWaitEvent(comm_s, ctx->ev[0], 0));
    // longest-first inside each part (a schedule only)
    int32_t *lpt = lpt_mode() ? dalloc<int32_t>(ctx, cw->nsegs) : nullptr;
    if (lpt) {
        ST(lpt_order(ctx, cw->seg_len, order, nloc, lpt));
        ST(lpt_order(ctx, cw->seg_len, order + nloc, nrem, lpt + nloc));
        dev_free(ctx, order, sizeof(int32_t) * cw->nsegs);
        order = lpt;
    }
    int pg = prof_begin(ctx, SPAMM_PH_GEMM);
    // the local segments leave exchange_ctas() SMs to the exchange's NCCL kernels (a
    // persistent GEMM CTA fills an SM's shared memory and most of its registers)
    ctx->gemm_grid_cap = std::max(1, ctx->sm_count - exchange_ctas());
    spamm_status st = gemm_run(ctx, cw, A, B, nullptr, m, epi, trace_part, order, nloc, 0);
    ctx->gemm_grid_cap = 0;
    prof_end(ctx, pg);
    // halo exchange with every allocation, kernel and collective on the comm stream
    double *halo = nullptr;
    int64_t nhalo = 0;
    if (!st) {
        ctx->stream = comm_s;
        int px = prof_begin(ctx, SPAMM_PH_OTHER);
        st = halo_exchange(ctx, cw, B, &halo, &nhalo);
        prof_end(ctx, px);
        ctx->stream = main_s;
        cw->stats.halo_blocks = nhalo;
        cw->stats.local_segments = nloc;
        cw->stats.transport = 1;
    }
    if (!st) {
        CK(cudaEventRecord(ctx->ev[1], comm_s));
        CK(cudaStreamWaitEvent(main_s, ctx->ev[1], 0));
        int pg2 = prof_begin(ctx, SPAMM_PH_GEMM);
        st = gemm_run(ctx, cw, A, B, halo, m, epi, trace_part, order + nloc, nrem, 1);
        prof_end(ctx, pg2);
        prof_gemm_work(ctx, cw->ntasks, cw->nsegs, A->b);
    }
    // self-check re-runs the GEMM while the halo (remote tiles, patched tB) still exists
    if (!st && selfcheck_mode()) selfcheck_gemm(ctx, cw, A, B, halo, m, epi);
    // the halo was allocated on the comm stream: free it there, after the GEMM read it
    CK(cudaEventRecord(ctx->ev[2], main_s));
    CK(cudaStreamWaitEvent(comm_s, ctx->ev[2], 0));
    ctx->stream = comm_s;
    dev_free(ctx, halo, sizeof(double) * nhalo * A->b * A->b);
    ctx->stream = main_s;
    dev_free(ctx, order, sizeof(int32_t) * cw->nsegs);
    return st;
}

// product with a given workspace and epilogue; C allocated here
// cull_done: the query already ran (cull_start + batched fetch + cull_complete);
// diag_dcount (EPI_NS_H only): append the absent diagonal blocks without a host round
// trip, their count lands there and the caller sets C->nblk after its next fetch.
static spamm_status product(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int epi,
                            double *trace_part, spamm_mat *C, int transA = 0, double alpha = 1.0,
                            bool cull_done = false, int64_t *diag_dcount = nullptr, double *t_out = nullptr)
{
    cw->alpha = alpha;
    if (transA && A->dist)
        return set_err(ctx, SPAMM_EINVAL, "A^T (x) B is not available on a row-partitioned context");
    if (A->dist != B->dist || A->r0 != B->r0 || A->r1 != B->r1)
        return set_err(ctx, SPAMM_ESHAPE, "operands have different row partitions");
    spamm_status sc = SPAMM_OK;
    if (!cull_done) {
        int pc = prof_begin(ctx, SPAMM_PH_CULL);
        sc = cull_run(ctx, cw, A, B, tau, A->r0, A->r1, transA);
        prof_end(ctx, pc);
        if (sc) return sc;
    }
    g_product_id++;
    if (selfcheck_mode()) selfcheck_cull(ctx, cw, A, B, tau, transA);
    if (ctx->vsink) ST(volume_record(ctx, cw));
    bool peer = false;
    if (A->dist && A->parts.world > 1) {
        int px = prof_begin(ctx, SPAMM_PH_OTHER);
        sc = peer_patch(ctx, cw, B, &peer);
        prof_end(ctx, px);
        if (sc) return sc;
    }
    // peer memory: one GEMM over all segments reading remote tiles in place; otherwise
    // the v2 halo exchange overlapped with the all-local segments
    const bool overlap = A->dist && A->parts.world > 1 && !peer;
    double *halo = nullptr;
    int64_t nhalo = 0;
    if (A->dist && !overlap && !peer) {
        // world size 1: nothing is remote, the exchange is a no-op
        int px = prof_begin(ctx, SPAMM_PH_OTHER);
        sc = halo_exchange(ctx, cw, B, &halo, &nhalo);
        prof_end(ctx, px);
        if (sc) return sc;
    }
    int64_t extra = (epi != EPI_STORE) ? A->nb : 0;
    spamm_mat m;
    spamm_status st = mat_new(ctx, A->n, A->b, cw->nsegs + extra, &m);
    if (!st && (m->r0 != A->r0 || m->r1 != A->r1)) {
        spamm_mat_free(m);
        st = set_err(ctx, SPAMM_EINVAL, "context partition changed since the operands were built");
    }
    if (st) {
        dev_free(ctx, halo, sizeof(double) * nhalo * A->b * A->b);
        if (peer) {   // the peers are waiting for this rank in the post-GEMM barrier
            cw->peer_world = 0;
            ctx->comm->peer_barrier(ctx);
        }
        return st;
    }
    st = mat_reset_pattern(ctx, m);
    if (!st && overlap) {
        // row partition, world > 1: the all-local segments run while the halo of remote
        // right-operand tiles is exchanged on the communication stream; then the rest
        st = overlapped_gemm(ctx, cw, A, B, m, epi, trace_part);
    } else if (!st) {
        int32_t *order = lpt_mode() ? dalloc<int32_t>(ctx, cw->nsegs) : nullptr;
        if (order) st = lpt_order(ctx, cw->seg_len, nullptr, cw->nsegs, order);
        int pg = prof_begin(ctx, SPAMM_PH_GEMM);
        if (!st) st = gemm_run(ctx, cw, A, B, halo, m, epi, trace_part, order, cw->nsegs, 0, transA);
        prof_end(ctx, pg);
        dev_free(ctx, order, sizeof(int32_t) * cw->nsegs);
        prof_gemm_work(ctx, cw->ntasks, cw->nsegs, A->b);
        if (!st && selfcheck_mode()) selfcheck_gemm(ctx, cw, A, B, halo, m, epi, transA);
    }
    dev_free(ctx, halo, sizeof(double) * nhalo * A->b * A->b);
    if (peer) {
        // every rank's reads of this rank's B are done before any rank goes on (and may
        // free or overwrite what it shared); the barrier runs whatever happened above
        cw->peer_world = 0;
        cw->stats.transport = 2;
        const spamm_status sb = ctx->comm->peer_barrier(ctx);
        if (!st) st = sb;
    }
    if (!st) {
        m->nblk = cw->nsegs;
        // absent diagonal blocks of X: H_ii = 1.5 I (plain map) or X_ii = 0 (scaled map,
        // mapped with the other blocks once alpha(t_k), eps(t_k) are known)
        if (epi == EPI_NS_H && diag_dcount)
            st = diag_fixup_async(ctx, m, cw->nsegs, 1.5, diag_dcount, t_out ? trace_part : nullptr, t_out);
        else if (epi == EPI_NS_H) st = diag_fixup(ctx, m, cw->nsegs, 1.5);
        if (epi == EPI_NS_X) st = diag_fixup(ctx, m, cw->nsegs, 0.0);
    }
    if (!st && epi != EPI_NS_X) st = norms_finish(ctx, m);
    if (st) {
        spamm_mat_free(m);
        return st;
    }
    *C = m;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_multiply(spamm_ctx ctx, spamm_mat A, spamm_mat B, double tau, spamm_mat *C,
                                       spamm_stats *stats)
{
    ST(check_pair(ctx, A, B, tau));
    if (!C) return set_err(ctx, SPAMM_EINVAL, "NULL output");
    ST(product(ctx, ctx->cw[0], A, B, tau, EPI_STORE, nullptr, C));
    if (stats) *stats = ctx->cw[0]->stats;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_multiply_t(spamm_ctx ctx, spamm_mat A, spamm_mat B, double tau, spamm_mat *C,
                                         spamm_stats *stats)
{
    ST(check_pair(ctx, A, B, tau));
    if (!C) return set_err(ctx, SPAMM_EINVAL, "NULL output");
    ST(product(ctx, ctx->cw[0], A, B, tau, EPI_STORE, nullptr, C, 1));
    if (stats) *stats = ctx->cw[0]->stats;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_export_tasks(spamm_ctx ctx, int32_t *ikj, int64_t cap, int64_t *n)
{
    if (!ctx || !n || (cap > 0 && !ikj)) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    if (!ctx->last) {
        *n = 0;
        return SPAMM_OK;
    }
    return cull_export(ctx, ctx->last, ikj, cap, n);
}

// The final unscale of spamm_ns_sqrt (Y * f, Z / f, f = sqrt(c (1+mu))) is fused into the
// Y' and Z' GEMM epilogues of the last step (saving a read + write pass over both results).
// The last step is known before those GEMMs run: k = iters - 1, or |t_k| <= t_stop with t_k
// from the X product of the same step.
struct FinalScale {
    bool force;      // last iteration by count
    double t_stop;   // > 0: also last when |t_k| <= t_stop
    double f;
    bool applied;    // out: Y', Z' were written unscaled
    // single device: the next step's X = Z' (x) Y' cull is enqueued before this step's
    // closing fetch and read back with it (one host round trip per step fewer)
    bool chain = false;        // in: a next step follows unless this one is the last
    bool x_ready = false;      // in: ctx->cw[0] already holds this step's X cull
    bool x_next_ready = false; // out: ctx->cw[0] holds the next step's X cull
};

// Single device: the step with three host round trips instead of five.  The X product
// appends H's absent diagonal blocks without reading their count back; then the Y' and
// Z' culls are both enqueued and ONE fetch brings back both queries' counters, the
// diagonal count, and t_k (which decides whether this is the last step, whose Y', Z'
// GEMMs carry the fused unscale).
static spamm_status ns_step_batched(spamm_ctx ctx, spamm_mat Y, spamm_mat Z, double tau, double tau_s, int32_t map,
                                    double *trace_part, spamm_mat *Hp, spamm_mat *Ynp, spamm_mat *Znp,
                                    spamm_stats stats[3], FinalScale *fs)
{
    const int nb = Y->nb;
    int64_t *ddiag = ctx->iscratch + 1;
    spamm_mat H = nullptr;
    // plain map: the trace t_k rides on the diagonal fix-up's launch
    spamm_status st = product(ctx, ctx->cw[0], Z, Y, tau, map ? EPI_NS_X : EPI_NS_H, trace_part, &H, 0, 1.0,
                              fs && fs->x_ready, map ? nullptr : ddiag, map ? nullptr : ctx->dscratch);
    const int64_t nseg = ctx->cw[0]->nsegs;
    if (!st && map) st = trace_finish(ctx, trace_part, nb, Y->n, ctx->dscratch);
    if (!st && map) st = ns_scaled_map(ctx, H, ctx->dscratch, ctx->dscratch + 8);
    if (!st && map) st = norms_finish(ctx, H);
    if (!st && stats) stats[0] = ctx->cw[0]->stats;
    Cull *c1 = ctx->cw[1], *c2 = ctx->cw[2];
    int pc = prof_begin(ctx, SPAMM_PH_CULL);
    // the Y' and Z' culls are independent, latency-bound chains of small kernels: the
    // Z' cull runs on the side stream, concurrently with the Y' cull
    const cudaStream_t main_s = ctx->stream;
    static const bool conc = [] {
        const char *e = getenv("SPAMM_CONCURRENT_CULL");
        return !(e && *e == '0');
    }();
    if (!st) st = ensure_side_stream(ctx);
    bool side_queued = false;   // work is queued on the side stream: it must be joined
    if (!st && !conc) {
        st = cull_start(ctx, c2, H, Z, tau, H->r0, H->r1);
    } else if (!st) {
        if (cudaEventRecord(ctx->ev[0], main_s) == cudaSuccess &&
            cudaStreamWaitEvent(ctx->comm_stream, ctx->ev[0], 0) == cudaSuccess) {
            side_queued = true;
            ctx->stream = ctx->comm_stream;
            st = cull_start(ctx, c2, H, Z, tau, H->r0, H->r1);
            ctx->stream = main_s;
        } else {
            st = set_err(ctx, SPAMM_ECUDA, "side stream fork");
        }
    }
    if (!st) st = cull_start(ctx, c1, Y, H, tau_s, Y->r0, Y->r1);
    // join the side stream whatever happened above: the caller frees H (whose pyramid
    // and slot map the side cull reads) with stream-ordered frees on main_s
    if (side_queued) {
        const bool joined = cudaEventRecord(ctx->ev[1], ctx->comm_stream) == cudaSuccess &&
                            cudaStreamWaitEvent(main_s, ctx->ev[1], 0) == cudaSuccess;
        if (!joined) {
            cudaStreamSynchronize(ctx->comm_stream);   // last resort: drain it from the host
            if (!st) st = set_err(ctx, SPAMM_ECUDA, "side stream join");
        }
    }
    int64_t added = 0;
    double tt = 0.0;
    if (!st) {
        FetchItem it[4] = {{c1->counters, c1->hcnt, 256}, {c2->counters, c2->hcnt, 256}, {ctx->dscratch, &tt, 8},
                           {ddiag, &added, 8}};
        st = fetch(ctx, it, map ? 3 : 4);
    }
    if (!st && !map) H->nblk = nseg + added;
    if (!st) st = cull_complete(ctx, c1, Y, H, tau_s, Y->r0, Y->r1);
    if (!st) st = cull_complete(ctx, c2, H, Z, tau, H->r0, H->r1);
    prof_end(ctx, pc);
    double ay = 1.0, az = 1.0;
    if (!st && fs && (fs->force || (fs->t_stop > 0.0 && std::fabs(tt) <= fs->t_stop))) {
        ay = fs->f;
        az = 1.0 / fs->f;
        fs->applied = true;
    }
    spamm_mat Yn = nullptr, Zn = nullptr;
    if (!st) st = product(ctx, c1, Y, H, tau_s, EPI_STORE, nullptr, &Yn, 0, ay, true);
    if (!st && stats) stats[1] = c1->stats;
    if (!st) st = product(ctx, c2, H, Z, tau, EPI_STORE, nullptr, &Zn, 0, az, true);
    if (!st && stats) stats[2] = c2->stats;
    *Hp = H;
    *Ynp = Yn;
    *Znp = Zn;
    return st;
}

static spamm_status ns_step_impl(spamm_ctx ctx, spamm_mat Y, spamm_mat Z, double tau, double tau_s, int32_t map,
                                 spamm_mat *Y_next, spamm_mat *Z_next, spamm_mat *H_out, double *t_k,
                                 spamm_stats stats[3], double *alpha_eps, FinalScale *fs)
{
    if (map != 0 && map != 1) return set_err(ctx, SPAMM_EINVAL, "map must be 0 or 1");
    ST(check_pair(ctx, Z, Y, tau));
    if (!(tau_s >= 0.0) || !std::isfinite(tau_s)) return set_err(ctx, SPAMM_EINVAL, "tau_s must be >= 0");
    if (!Y_next || !Z_next) return set_err(ctx, SPAMM_EINVAL, "NULL output");
    const int nb = Y->nb;
    double *trace_part = dalloc<double>(ctx, nb);
    if (!trace_part) return set_err(ctx, SPAMM_ENOMEM, "trace partials");
    CK(cudaMemsetAsync(trace_part, 0, sizeof(double) * nb, ctx->stream));
    spamm_mat H = nullptr, Yn = nullptr, Zn = nullptr;
    if (!Y->dist) {
        spamm_status sb = ns_step_batched(ctx, Y, Z, tau, tau_s, map, trace_part, &H, &Yn, &Zn, stats, fs);
        double hv[3] = {0, 0, 0}, ae[2] = {1.0, 0.0};
        // the next step's X cull rides on this step's closing fetch (wasted only if the
        // step turns out non-finite)
        const bool chain = !sb && fs && fs->chain && !fs->applied;
        if (chain) {
            int pc = prof_begin(ctx, SPAMM_PH_CULL);
            sb = cull_start(ctx, ctx->cw[0], Zn, Yn, tau, Zn->r0, Zn->r1);
            prof_end(ctx, pc);
        }
        if (!sb) {
            FetchItem it[5] = {{ctx->dscratch, &hv[0], 8}, {Yn->norm2, &hv[1], 8}, {Zn->norm2, &hv[2], 8},
                               {ctx->dscratch + 8, ae, 16}, {ctx->cw[0]->counters, ctx->cw[0]->hcnt, 256}};
            if (chain && !map) it[3] = it[4];
            sb = fetch(ctx, it, 3 + (map ? 1 : 0) + (chain ? 1 : 0));
        }
        if (!sb && chain && std::isfinite(hv[0]) && std::isfinite(hv[1]) && std::isfinite(hv[2])) {
            sb = cull_complete(ctx, ctx->cw[0], Zn, Yn, tau, Zn->r0, Zn->r1);
            if (!sb) fs->x_next_ready = true;
        }
        dev_free(ctx, trace_part, sizeof(double) * nb);
        if (sb) {
            spamm_mat_free(H);
            spamm_mat_free(Yn);
            spamm_mat_free(Zn);
            return sb;
        }
        if (t_k) *t_k = hv[0];
        if (alpha_eps) {
            alpha_eps[0] = ae[0];
            alpha_eps[1] = ae[1];
        }
        if (H_out) *H_out = H;
        else spamm_mat_free(H);
        *Y_next = Yn;
        *Z_next = Zn;
        if (!std::isfinite(hv[0]) || !std::isfinite(hv[1]) || !std::isfinite(hv[2]))
            return set_err(ctx, SPAMM_ENOTFINITE, "non-finite trace error or root norm");
        return SPAMM_OK;
    }
    // X = Z (x)_tau Y  ->  H = 1/2 (3I - X), tr X partials (X never stored); scaled map:
    // X stored, then H = h_alpha[(1-2eps)X + eps I] in place once t_k is known
    spamm_status st = product(ctx, ctx->cw[0], Z, Y, tau, map ? EPI_NS_X : EPI_NS_H, trace_part, &H);
    // row partition: every rank gets all tr(X_ii) partials, summed in the fixed order
    if (!st && H->dist) st = gather_rows(ctx, H->parts, trace_part, 1);
    if (!st) st = trace_finish(ctx, trace_part, nb, Y->n, ctx->dscratch);
    if (!st && map) st = ns_scaled_map(ctx, H, ctx->dscratch, ctx->dscratch + 8);
    if (!st && map) st = norms_finish(ctx, H);
    if (!st && stats) stats[0] = ctx->cw[0]->stats;
    double ay = 1.0, az = 1.0;
    if (!st && fs) {
        bool last = fs->force;
        if (!last && fs->t_stop > 0.0) {
            double tt = 0.0;
            st = fetch1(ctx, ctx->dscratch, &tt, sizeof(double));
            last = !st && std::fabs(tt) <= fs->t_stop;
        }
        if (last) {
            ay = fs->f;
            az = 1.0 / fs->f;
            fs->applied = true;
        }
    }
    // Y' = Y (x)_tau_s H ; Z' = H (x)_tau Z
    if (!st) st = product(ctx, ctx->cw[1], Y, H, tau_s, EPI_STORE, nullptr, &Yn, 0, ay);
    if (!st && stats) stats[1] = ctx->cw[1]->stats;
    if (!st) st = product(ctx, ctx->cw[2], H, Z, tau, EPI_STORE, nullptr, &Zn, 0, az);
    if (!st && stats) stats[2] = ctx->cw[2]->stats;
    double hv[3] = {0, 0, 0}, ae[2] = {1.0, 0.0};
    if (!st) {
        // t_k and the root norms (non-finite detection)
        FetchItem it[4] = {{ctx->dscratch, &hv[0], 8}, {Yn->norm2, &hv[1], 8}, {Zn->norm2, &hv[2], 8},
                           {ctx->dscratch + 8, ae, 16}};
        st = fetch(ctx, it, map ? 4 : 3);
    }
    dev_free(ctx, trace_part, sizeof(double) * nb);
    if (st) {
        spamm_mat_free(H);
        spamm_mat_free(Yn);
        spamm_mat_free(Zn);
        return st;
    }
    if (t_k) *t_k = hv[0];
    if (alpha_eps) {
        alpha_eps[0] = ae[0];
        alpha_eps[1] = ae[1];
    }
    if (H_out) *H_out = H;
    else spamm_mat_free(H);
    *Y_next = Yn;
    *Z_next = Zn;
    if (!std::isfinite(hv[0]) || !std::isfinite(hv[1]) || !std::isfinite(hv[2]))
        return set_err(ctx, SPAMM_ENOTFINITE, "non-finite trace error or root norm");
    return SPAMM_OK;
}

extern "C" spamm_status spamm_ns_step_map(spamm_ctx ctx, spamm_mat Y, spamm_mat Z, double tau, double tau_s,
                                          int32_t map, spamm_mat *Y_next, spamm_mat *Z_next, spamm_mat *H_out,
                                          double *t_k, spamm_stats stats[3], double *alpha_eps)
{
    return ns_step_impl(ctx, Y, Z, tau, tau_s, map, Y_next, Z_next, H_out, t_k, stats, alpha_eps, nullptr);
}

extern "C" spamm_status spamm_ns_step(spamm_ctx ctx, spamm_mat Y, spamm_mat Z, double tau, double tau_s,
                                      spamm_mat *Y_next, spamm_mat *Z_next, spamm_mat *H_out,
                                      double *t_k, spamm_stats stats[3])
{
    return spamm_ns_step_map(ctx, Y, Z, tau, tau_s, 0, Y_next, Z_next, H_out, t_k, stats, nullptr);
}

extern "C" spamm_status spamm_power_scale(spamm_ctx ctx, spamm_mat s, int32_t K, double *c)
{
    if (!ctx || !s || !c || K < 0) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    return power_scale(ctx, s, K, c);
}

// ------------------------------------------------ graph-replayed NS steps
// Small problems are latency-bound (C1: ~25 launches and 2 host round trips per step
// for ~1 MFLOP).  When the worst-case workspace fits a memory budget, the dual step is
// made device-driven and captured once as a CUDA graph:
//   * every capacity is the worst case (cull levels <= nb^3 triples, segments and
//     output blocks <= nb^2), so nothing can overflow and no count is needed on the host;
//   * the GEMMs read their segment count from the cull's counters, the diagonal
//     fix-up its base slot; grids are capacity-sized (the kernels loop over their work);
//   * matrices ping-pong between two fixed buffer sets (Y_k, Z_k) -> (Y_k+1, Z_k+1);
//   * a record kernel appends t_k, the three products' level counts and the root
//     norms of Y', Z' to a device log, read once after the last replay.
// Same kernels, same arguments, same orders as the host-driven step: the results are
// bitwise those of the classic path (tests/test_gpu_determinism.py).  The last step
// (fused final unscale) runs host-driven.  Any non-finite value in the log sends the
// whole run back to the host-driven loop (which stops at the failing step).
struct StepRec {
    double t, ny2, nz2, pad;
    int32_t cnt[3][20];   // per product: level counts [0..15], overflow [16], segments [17]
};

__global__ void k_step_record(double *t_dev, const int32_t *c0, const int32_t *c1, const int32_t *c2,
                              const double *ny2, const double *nz2, StepRec *rec, int32_t *k)
{
    pdl_wait();
    const int i = *k;
    StepRec &r = rec[i];
    const int32_t *c[3] = {c0, c1, c2};
    for (int e = threadIdx.x; e < 60; e += blockDim.x) r.cnt[e / 20][e % 20] = c[e / 20][e % 20];
    if (threadIdx.x == 0) {
        r.t = *t_dev;
        r.ny2 = *ny2;
        r.nz2 = *nz2;
        r.pad = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) *k = i + 1;
}

struct NsGraph {
    int64_t n = 0;
    int b = 0;
    double tau = -1.0, tau_s = -1.0;
    spamm_mat Yb[2] = {nullptr, nullptr}, Zb[2] = {nullptr, nullptr}, H = nullptr;
    double *trace_part = nullptr;
    int32_t *newslot = nullptr;
    int64_t *hadd = nullptr;
    StepRec *rec = nullptr;
    int rec_cap = 0;
    int32_t *kdev = nullptr;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    int64_t kernels[2] = {0, 0};
    int64_t gen[3] = {-1, -1, -1};
};

static void ns_graph_free(spamm_ctx ctx)
{
    NsGraph *g = ctx->nsg;
    if (!g) return;
    cudaStreamSynchronize(ctx->stream);
    for (auto &e : g->exec)
        if (e) cudaGraphExecDestroy(e);
    for (spamm_mat m : {g->Yb[0], g->Yb[1], g->Zb[0], g->Zb[1], g->H}) spamm_mat_free(m);
    const int nb = (int)(g->b ? g->n / g->b : 0);
    dev_free(ctx, g->trace_part, sizeof(double) * nb);
    dev_free(ctx, g->newslot, sizeof(int32_t) * nb);
    dev_free(ctx, g->hadd, sizeof(int64_t));
    dev_free(ctx, g->rec, sizeof(StepRec) * g->rec_cap);
    dev_free(ctx, g->kdev, sizeof(int32_t));
    delete g;
    ctx->nsg = nullptr;
}

// SPAMM_GRAPH: 0 = off, 1 = auto (worst case <= 4 GiB, default), 2 = up to 32 GiB
static int graph_mode()
{
    static const int m = [] {
        const char *e = getenv("SPAMM_GRAPH");
        return e && *e ? atoi(e) : 1;
    }();
    return m;
}

static bool ns_graph_eligible(spamm_ctx ctx, spamm_mat s, const spamm_ns_opts &o, int iters)
{
    const int gm = graph_mode();
    if (!gm || s->dist || o.map != 0 || o.t_stop > 0.0 || iters < 2 || ctx->vsink || selfcheck_mode() ||
        lpt_mode())
        return false;
    const double nb = (double)s->nb, b2 = (double)s->b * s->b;
    const double mats = 5.0 * (nb * nb * (8.0 * b2 + 8.0) + 8.0 * (double)pyr_size(s->L));
    const double culls = 3.0 * nb * nb * nb * 61.0;
    return mats + culls <= (gm >= 2 ? 32.0 : 4.0) * (1u << 30);
}

// SPAMM_GRAPH_SPLIT: 0 = Y', Z' GEMMs one after the other on all SMs, 2 = concurrently on
// half the SMs each, 1 (default) = concurrently only for nb <= 32 (C1: GEMMs of ~100
// segments; at C2, ~1000 segments each, the full grid wins: 3.9 vs 5.0 ms per run)
static bool graph_split(int nb)
{
    static const int m = [] {
        const char *e = getenv("SPAMM_GRAPH_SPLIT");
        return e && *e ? atoi(e) : 1;
    }();
    return m == 2 || (m == 1 && nb <= 32);
}

// SPAMM_GRAPH_SIDE_CLEAR=0: the pattern clearing inside the X cull's (single-CTA) kernel
static bool graph_side_clear()
{
    static const int m = [] {
        const char *e = getenv("SPAMM_GRAPH_SIDE_CLEAR");
        return e && *e ? atoi(e) : 1;
    }();
    return m != 0;
}

// SPAMM_GRAPH_PAIR=0: the Y' and Z' GEMMs (and pyramids) as separate launches (A/B runs)
static bool graph_pair()
{
    static const int m = [] {
        const char *e = getenv("SPAMM_GRAPH_PAIR");
        return e && *e ? atoi(e) : 1;
    }();
    return m != 0;
}

// One device-driven dual step: (Y, Z) -> (Yn, Zn) through the fixed buffers (captured).
//   main:  X cull (also clears H, Y', Z' patterns and the trace partials) -> X GEMM ->
//          diagonal fix-up -> pyramid(H) -> t_k -> fork
//   main:  Y' cull [-> Y' GEMM (half the SMs) -> pyramid(Y')]   } concurrent branches
//   side:  Z' cull [-> Z' GEMM (half the SMs) -> pyramid(Z')]   } ([..]: split mode)
//   join [-> Y' and Z' GEMMs in one launch -> both pyramids in one launch] -> step record.
// For nb >= 64 the H, Y', Z' pattern clearing runs on the side stream beside the X cull.
static spamm_status graph_step(spamm_ctx ctx, NsGraph *g, spamm_mat Y, spamm_mat Z, spamm_mat Yn, spamm_mat Zn)
{
    Cull *c0 = ctx->cw[0], *c1 = ctx->cw[1], *c2 = ctx->cw[2];
    spamm_mat H = g->H;
    const int nb = Y->nb;
    CullClear clr{{H->slot, Yn->slot, Zn->slot}, {H->norm2, Yn->norm2, Zn->norm2}, (int64_t)nb * nb,
                  pyr_size(Y->L), g->trace_part, nb};
    // X = Z (x)_tau Y -> H = 1/2 (3I - X), tr X partials, absent diagonal blocks 1.5 I.  The
    // H, Y', Z' patterns are cleared by a kernel on the side stream beside the X cull (they are
    // none of its inputs); the X GEMM, which writes H, waits for it.
    if (graph_side_clear() && nb >= 64) {   // (C1, nb = 16: the fork costs more than the clear)
        CK(cudaEventRecord(ctx->ev[2], ctx->stream));
        CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev[2], 0));
        const cudaStream_t ms = ctx->stream;
        ctx->stream = ctx->comm_stream;
        const spamm_status cs = cull_clear_enqueue(ctx, clr);
        ctx->stream = ms;
        ST(cs);
        CK(cudaEventRecord(ctx->ev[2], ctx->comm_stream));
        ST(cull_enqueue_fixed(ctx, c0, Z, Y, g->tau, nullptr));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev[2], 0));
    } else {
        ST(cull_enqueue_fixed(ctx, c0, Z, Y, g->tau, &clr));
    }
    c0->alpha = 1.0;
    ST(gemm_run(ctx, c0, Z, Y, nullptr, H, EPI_NS_H, g->trace_part, nullptr, 0, 0, 0, true));
    ST(diag_fixup_dev(ctx, H, c0->counters + CNT_NSEG, 1.5, g->newslot, g->hadd, g->trace_part, ctx->dscratch));
    ST(pyramid_build(ctx, H));
    // Y' = Y (x)_tau_s H on the main stream || Z' = H (x)_tau Z on the side stream: the two
    // culls always; with split, the GEMMs (each on half the SMs) and pyramids as well
    const bool split = graph_split(nb);
    const cudaStream_t main_s = ctx->stream;
    CK(cudaEventRecord(ctx->ev[0], main_s));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev[0], 0));
    c1->alpha = c2->alpha = 1.0;
    if (split) ctx->gemm_grid_cap = std::max(1, ctx->sm_count / 2);
    ctx->stream = ctx->comm_stream;
    spamm_status st = cull_enqueue_fixed(ctx, c2, H, Z, g->tau);
    if (!st && split) st = gemm_run(ctx, c2, H, Z, nullptr, Zn, EPI_STORE, nullptr, nullptr, 0, 0, 0, true);
    if (!st && split) st = pyramid_build(ctx, Zn);
    ctx->stream = main_s;
    if (!st) st = cull_enqueue_fixed(ctx, c1, Y, H, g->tau_s);
    if (!st && split) st = gemm_run(ctx, c1, Y, H, nullptr, Yn, EPI_STORE, nullptr, nullptr, 0, 0, 0, true);
    if (!st && split) st = pyramid_build(ctx, Yn);
    ctx->gemm_grid_cap = 0;
    ST(st);
    CK(cudaEventRecord(ctx->ev[1], ctx->comm_stream));
    CK(cudaStreamWaitEvent(main_s, ctx->ev[1], 0));
    if (!split && graph_pair()) {
        // Y' and Z' in one GEMM launch (tickets over both segment lists) and their pyramids in
        // one launch per pass: two launch boundaries fewer on the step's critical path
        ST(gemm_run_pair(ctx, c1, Y, H, Yn, c2, H, Z, Zn));
        ST(pyramid_build_pair(ctx, Yn, Zn));
    } else if (!split) {
        ST(gemm_run(ctx, c1, Y, H, nullptr, Yn, EPI_STORE, nullptr, nullptr, 0, 0, 0, true));
        ST(pyramid_build(ctx, Yn));
        ST(gemm_run(ctx, c2, H, Z, nullptr, Zn, EPI_STORE, nullptr, nullptr, 0, 0, 0, true));
        ST(pyramid_build(ctx, Zn));
    }
    CK(launch_pdl(k_step_record, 1, 64, 0, ctx->stream, ctx->dscratch, (const int32_t *)c0->counters,
                  (const int32_t *)c1->counters, (const int32_t *)c2->counters, (const double *)Yn->norm2,
                  (const double *)Zn->norm2, g->rec, g->kdev));
    CKL(ctx);
    return SPAMM_OK;
}

static spamm_status ns_graph_prepare(spamm_ctx ctx, spamm_mat s, double tau, double tau_s, int steps)
{
    NsGraph *g = ctx->nsg;
    const int64_t nb = s->nb;
    const bool same = g && g->n == s->n && g->b == s->b && g->tau == tau && g->tau_s == tau_s;
    if (!same) {
        ns_graph_free(ctx);
        g = ctx->nsg = new NsGraph();
        g->n = s->n;
        g->b = s->b;
        g->tau = tau;
        g->tau_s = tau_s;
        spamm_mat *all[5] = {&g->Yb[0], &g->Yb[1], &g->Zb[0], &g->Zb[1], &g->H};
        for (spamm_mat *m : all) ST(mat_new(ctx, s->n, s->b, nb * nb, m));
        g->trace_part = dalloc<double>(ctx, nb);
        g->newslot = dalloc<int32_t>(ctx, nb);
        g->hadd = dalloc<int64_t>(ctx, 1);
        g->kdev = dalloc<int32_t>(ctx, 1);
        if (!g->trace_part || !g->newslot || !g->hadd || !g->kdev) return set_err(ctx, SPAMM_ENOMEM, "graph state");
    }
    if (g->rec_cap < steps) {
        dev_free(ctx, g->rec, sizeof(StepRec) * g->rec_cap);
        g->rec_cap = std::max(steps, 64);
        g->rec = dalloc<StepRec>(ctx, g->rec_cap);
        if (!g->rec) {
            g->rec_cap = 0;
            return set_err(ctx, SPAMM_ENOMEM, "graph log");
        }
        for (auto &e : g->exec)   // the log pointer is baked into the graphs
            if (e) {
                cudaGraphExecDestroy(e);
                e = nullptr;
            }
    }
    for (int i = 0; i < 3; i++) {
        ST(cull_reserve(ctx, ctx->cw[i], nb * nb * nb, nb * nb));
        if (ctx->cw[i]->gen != g->gen[i]) {
            for (auto &e : g->exec)
                if (e) {
                    cudaGraphExecDestroy(e);
                    e = nullptr;
                }
        }
    }
    ST(ensure_side_stream(ctx));
    for (int p = 0; p < 2; p++) {
        if (g->exec[p]) continue;
        for (int i = 0; i < 3; i++) ctx->cw[i]->prevL = -1;
        const int64_t l0 = ctx->launches;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        ctx->capturing = true;
        spamm_status st = graph_step(ctx, g, g->Yb[p], g->Zb[p], g->Yb[p ^ 1], g->Zb[p ^ 1]);
        ctx->capturing = false;
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
        g->kernels[p] = ctx->launches - l0;
        ctx->launches = l0;
        if (st) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return check_cuda(ctx, e, "graph capture");
        e = cudaGraphInstantiate(&g->exec[p], graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            g->exec[p] = nullptr;
            return check_cuda(ctx, e, "graph instantiate");
        }
    }
    for (int i = 0; i < 3; i++) g->gen[i] = ctx->cw[i]->gen;
    return SPAMM_OK;
}

static spamm_status mat_copy_into(spamm_ctx ctx, spamm_mat dst, spamm_mat src)
{
    const int64_t nb = src->nb;
    CK(cudaMemcpyAsync(dst->norm2, src->norm2, sizeof(double) * pyr_size(src->L), cudaMemcpyDeviceToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(dst->slot, src->slot, sizeof(int32_t) * nb * nb, cudaMemcpyDeviceToDevice, ctx->stream));
    if (src->nblk > 0) {
        CK(cudaMemcpyAsync(dst->pool, src->pool, sizeof(double) * src->nblk * src->b * src->b,
                           cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(dst->coord, src->coord, sizeof(int32_t) * src->nblk, cudaMemcpyDeviceToDevice,
                           ctx->stream));
    }
    dst->nblk = src->nblk;
    return SPAMM_OK;
}

static void rec_stats(const StepRec &r, int L, int b, spamm_stats *out)
{
    const int l0 = L < 4 ? L : 4;   // cull.cu INIT_L0
    for (int p = 0; p < 3; p++) {
        spamm_stats &s = out[p];
        s = spamm_stats{};
        s.tasks = r.cnt[p][L];
        s.segments = r.cnt[p][CNT_NSEG];
        for (int l = l0; l <= L && l < 24; l++) s.level_survivors[l] = r.cnt[p][l];
        s.candidates = L > l0 ? 8 * (int64_t)r.cnt[p][L - 1] : ((int64_t)1 << (3 * L));
        s.flops = 2.0 * (double)b * b * b * (double)s.tasks;
    }
}

// Runs `steps` dual steps from (Y, Z) by graph replay.  On success *Yk, *Zk are the
// context's buffers holding (Y_steps, Z_steps) (borrowed: owned by ctx->nsg) and the
// history is filled; *ok = false (and SPAMM_OK) when the log shows a non-finite value
// or an overflow: the caller redoes the run host-driven.
static spamm_status ns_graph_run(spamm_ctx ctx, spamm_mat Y, spamm_mat Z, double tau, double tau_s, int steps,
                                 const spamm_ns_opts &o, spamm_mat *Yk, spamm_mat *Zk, bool *ok)
{
    *ok = false;
    ST(ns_graph_prepare(ctx, Y, tau, tau_s, steps));
    NsGraph *g = ctx->nsg;
    ST(mat_copy_into(ctx, g->Yb[0], Y));
    ST(mat_copy_into(ctx, g->Zb[0], Z));
    CK(cudaMemsetAsync(g->kdev, 0, sizeof(int32_t), ctx->stream));
    for (int k = 0; k < steps; k++) {
        CK(cudaGraphLaunch(g->exec[k & 1], ctx->stream));
        ctx->launches += g->kernels[k & 1];
    }
    std::vector<StepRec> rec(steps);
    CK(cudaMemcpyAsync(rec.data(), g->rec, sizeof(StepRec) * steps, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const int L = Y->L, b = Y->b;
    for (int k = 0; k < steps; k++) {
        const StepRec &r = rec[k];
        if (!std::isfinite(r.t) || !std::isfinite(r.ny2) || !std::isfinite(r.nz2)) return SPAMM_OK;
        for (int p = 0; p < 3; p++)
            if (r.cnt[p][CNT_OVERFLOW]) return SPAMM_OK;
    }
    for (int k = 0; k < steps; k++) {
        spamm_stats st[3];
        rec_stats(rec[k], L, b, st);
        if (o.t_history) o.t_history[k] = rec[k].t;
        if (o.per_product) memcpy(o.per_product + 3 * k, st, sizeof(st));
        // (no prof_gemm_work: the graph's GEMMs carry no phase events, so the GEMM
        // roofline of a profiled run covers the host-driven products only)
    }
    const int q = steps & 1;
    g->Yb[q]->nblk = rec[steps - 1].cnt[1][CNT_NSEG];
    g->Zb[q]->nblk = rec[steps - 1].cnt[2][CNT_NSEG];
    *Yk = g->Yb[q];
    *Zk = g->Zb[q];
    *ok = true;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_ns_sqrt(spamm_ctx ctx, spamm_mat s, double tau, int32_t iters, spamm_mat *Yout,
                                      spamm_mat *Zout, const spamm_ns_opts *opts)
{
    if (!ctx || !s || !Yout || !Zout) return set_err(ctx, SPAMM_EINVAL, "NULL argument");
    if (iters < 1) return set_err(ctx, SPAMM_EINVAL, "iters must be >= 1");
    if (!(tau >= 0.0) || !std::isfinite(tau)) return set_err(ctx, SPAMM_EINVAL, "tau must be finite and >= 0");
    spamm_ns_opts o{};
    o.tau_s = -1.0;
    o.power_iters = 100;
    if (opts) o = *opts;
    if (o.power_iters <= 0) o.power_iters = 100;
    double tau_s = o.tau_s < 0.0 ? tau : o.tau_s;
    double mu = o.mu;
    if (!(mu >= 0.0)) return set_err(ctx, SPAMM_EINVAL, "mu must be >= 0");
    int ps = prof_begin(ctx, SPAMM_PH_SETUP);
    double root = 0.0;
    ST(spamm_norm(ctx, s, &root));
    if (!(root > 0.0)) return set_err(ctx, SPAMM_EINVAL, "s is zero");
    double c = o.scale;
    if (!(c > 0.0)) ST(power_scale(ctx, s, o.power_iters, &c));
    if (o.c_out) *o.c_out = c;
    if (o.iters_done) *o.iters_done = 0;
    spamm_mat Y = nullptr, Z = nullptr;
    ST(spamm_ns_y0(ctx, s, c, mu, &Y));
    spamm_status st = spamm_identity(ctx, s->n, s->b, &Z);
    prof_end(ctx, ps);
    int pl = prof_begin(ctx, SPAMM_PH_LOOP);
    const double f = std::sqrt(c * (1.0 + mu));
    bool unscaled = false;   // Y, Z already hold the outputs (final unscale fused)
    bool x_ready = false;    // ctx->cw[0] holds the coming step's X cull (chained fetch)
    bool borrowed = false;   // Y, Z are the graph's buffers (not freed here)
    int k0 = 0;
    if (!st && ns_graph_eligible(ctx, s, o, iters)) {
        spamm_mat Yk = nullptr, Zk = nullptr;
        bool ok = false;
        st = ns_graph_run(ctx, Y, Z, tau, tau_s, iters - 1, o, &Yk, &Zk, &ok);
        if (!st && ok) {
            spamm_mat_free(Y);
            spamm_mat_free(Z);
            Y = Yk;
            Z = Zk;
            borrowed = true;
            k0 = iters - 1;
            if (o.iters_done) *o.iters_done = k0;
        }
    }
    for (int k = k0; k < iters && !st; k++) {
        spamm_mat Yn = nullptr, Zn = nullptr;
        double t = 0.0;
        spamm_stats sts[3];
        FinalScale fs{k == iters - 1, o.t_stop, f, false};
        fs.chain = k + 1 < iters;
        fs.x_ready = x_ready;
        st = ns_step_impl(ctx, Y, Z, tau, tau_s, o.map, &Yn, &Zn, nullptr, &t, sts, nullptr, &fs);
        x_ready = fs.x_next_ready;
        if (o.t_history && (st == SPAMM_OK || st == SPAMM_ENOTFINITE)) o.t_history[k] = t;
        if (o.per_product && st == SPAMM_OK) memcpy(o.per_product + 3 * k, sts, sizeof(sts));
        if (st) {
            spamm_mat_free(Yn);
            spamm_mat_free(Zn);
            break;
        }
        if (!borrowed) {
            spamm_mat_free(Y);
            spamm_mat_free(Z);
        }
        borrowed = false;
        Y = Yn;
        Z = Zn;
        unscaled = fs.applied;
        if (o.iters_done) *o.iters_done = k + 1;
        if (unscaled) break;   // the last step (by count or by |t_k| <= t_stop)
    }
    prof_end(ctx, pl);
    std::string err = ctx->err;
    spamm_status st2 = SPAMM_OK;
    if (Y && Z && borrowed) {
        // a failure right after the graph steps: hand out copies, the buffers stay cached
        spamm_mat Yf = nullptr, Zf = nullptr;
        st2 = mat_map(ctx, Y, 2, f, 0.0, &Yf);
        if (!st2) st2 = mat_map(ctx, Z, 0, f, 0.0, &Zf);
        if (!st2) {
            *Yout = Yf;
            *Zout = Zf;
        } else {
            spamm_mat_free(Yf);
            spamm_mat_free(Zf);
        }
    } else if (Y && Z && unscaled) {
        *Yout = Y;
        *Zout = Z;
    } else if (Y && Z) {
        // unscale: Y * sqrt(c(1+mu)) -> (s + c mu I)^{1/2}, Z / sqrt(c(1+mu)) -> (s + c mu I)^{-1/2}
        spamm_mat Yf = nullptr, Zf = nullptr;
        st2 = mat_map(ctx, Y, 2, f, 0.0, &Yf);
        if (!st2) st2 = mat_map(ctx, Z, 0, f, 0.0, &Zf);
        spamm_mat_free(Y);
        spamm_mat_free(Z);
        if (!st2) {
            *Yout = Yf;
            *Zout = Zf;
        } else {
            spamm_mat_free(Yf);
            spamm_mat_free(Zf);
        }
    }
    if (st) {
        ctx->err = err;
        return st;
    }
    return st2;
}

// ------------------------------------------------------------ single channel
// PAPER.md Eq. single, sensitive product rightmost:
//   Z_{k+1} = Z_k (x)_tau H_k,  W_{k+1} = s' (x)_tau_s Z_{k+1},
//   H_{k+1} = h[Z_{k+1}^T (x)_tau W_{k+1}]  (X never stored for the plain map),
// s' = s/c, Z_0 = I, X_0 = s' (t_0, H_0 = h[X_0] by maps), outputs Z -> s^{-1/2},
// Y = W sqrt(c) -> s^{1/2}.  Not available on a row-partitioned context (Z^T).

// t = (n - tr m)/n from the stored diagonal blocks (fixed order per block, then
// the fixed-order trace_finish)
__global__ void k_diag_trace(const double *pool, const int32_t *slot, int nb, int b, double *part)
{
    const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= nb) return;
    const int s = slot[morton(i, i)];
    double t = 0.0;
    if (s >= 0)
        for (int r = lane; r < b; r += 32) t += pool[(int64_t)s * b * b + pool_at(r, r, b)];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) part[i] = t;
}

static spamm_status mat_trace_err(spamm_ctx ctx, spamm_mat m, double *t_dev)
{
    double *part = dalloc<double>(ctx, m->nb);
    if (!part) return set_err(ctx, SPAMM_ENOMEM, "trace");
    k_diag_trace<<<cdiv(m->nb, 8), 256, 0, ctx->stream>>>(m->pool, m->slot, m->nb, m->b, part);
    CKL(ctx);
    spamm_status st = trace_finish(ctx, part, m->nb, m->n, t_dev);
    dev_free(ctx, part, sizeof(double) * m->nb);
    return st;
}

// H = h[X] of a stored X by maps (the initial H_0 = h[s']): t from the trace first
static spamm_status h_of(spamm_ctx ctx, spamm_mat X, int map, spamm_mat *H)
{
    ST(mat_trace_err(ctx, X, ctx->dscratch));
    if (!map) return mat_map(ctx, X, 4, 0.0, 0.0, H);
    spamm_mat C;
    ST(mat_map(ctx, X, 7, 0.0, 0.0, &C));
    spamm_status st = ns_scaled_map(ctx, C, ctx->dscratch, ctx->dscratch + 8);
    if (!st) st = norms_finish(ctx, C);
    if (st) {
        spamm_mat_free(C);
        return st;
    }
    *H = C;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_ns_step_single(spamm_ctx ctx, spamm_mat S1, spamm_mat Z, spamm_mat H, double tau,
                                             double tau_s, int32_t map, spamm_mat *Z_next, spamm_mat *H_next,
                                             spamm_mat *W_out, double *t_next, spamm_stats stats[3],
                                             double *alpha_eps)
{
    ST(check_pair(ctx, Z, H, tau));
    ST(check_pair(ctx, S1, Z, tau));
    if (!(tau_s >= 0.0) || !std::isfinite(tau_s)) return set_err(ctx, SPAMM_EINVAL, "tau_s must be >= 0");
    if (map != 0 && map != 1) return set_err(ctx, SPAMM_EINVAL, "map must be 0 or 1");
    if (!Z_next || !H_next) return set_err(ctx, SPAMM_EINVAL, "NULL output");
    if (Z->dist) return set_err(ctx, SPAMM_EINVAL, "single channel needs Z^T: not on a row-partitioned context");
    const int nb = Z->nb;
    double *trace_part = dalloc<double>(ctx, nb);
    if (!trace_part) return set_err(ctx, SPAMM_ENOMEM, "trace partials");
    CK(cudaMemsetAsync(trace_part, 0, sizeof(double) * nb, ctx->stream));
    spamm_mat Zn = nullptr, W = nullptr, Hn = nullptr;
    spamm_status st = product(ctx, ctx->cw[0], Z, H, tau, EPI_STORE, nullptr, &Zn);
    if (!st && stats) stats[0] = ctx->cw[0]->stats;
    if (!st) st = product(ctx, ctx->cw[1], S1, Zn, tau_s, EPI_STORE, nullptr, &W);
    if (!st && stats) stats[1] = ctx->cw[1]->stats;
    if (!st) st = product(ctx, ctx->cw[2], Zn, W, tau, map ? EPI_NS_X : EPI_NS_H, trace_part, &Hn, 1);
    if (!st && stats) stats[2] = ctx->cw[2]->stats;
    if (!st) st = trace_finish(ctx, trace_part, nb, Z->n, ctx->dscratch);
    if (!st && map) st = ns_scaled_map(ctx, Hn, ctx->dscratch, ctx->dscratch + 8);
    if (!st && map) st = norms_finish(ctx, Hn);
    double hv[3] = {0, 0, 0}, ae[2] = {1.0, 0.0};
    if (!st) {
        FetchItem it[4] = {{ctx->dscratch, &hv[0], 8}, {Zn->norm2, &hv[1], 8}, {Hn->norm2, &hv[2], 8},
                           {ctx->dscratch + 8, ae, 16}};
        st = fetch(ctx, it, map ? 4 : 3);
    }
    dev_free(ctx, trace_part, sizeof(double) * nb);
    if (st) {
        spamm_mat_free(Zn);
        spamm_mat_free(W);
        spamm_mat_free(Hn);
        return st;
    }
    if (t_next) *t_next = hv[0];
    if (alpha_eps) {
        alpha_eps[0] = ae[0];
        alpha_eps[1] = ae[1];
    }
    *Z_next = Zn;
    *H_next = Hn;
    if (W_out) *W_out = W;
    else spamm_mat_free(W);
    if (!std::isfinite(hv[0]) || !std::isfinite(hv[1]) || !std::isfinite(hv[2]))
        return set_err(ctx, SPAMM_ENOTFINITE, "non-finite trace error or root norm");
    return SPAMM_OK;
}

extern "C" spamm_status spamm_ns_sqrt_single(spamm_ctx ctx, spamm_mat s, double tau, int32_t iters,
                                             spamm_mat *Yout, spamm_mat *Zout, const spamm_ns_opts *opts)
{
    if (!ctx || !s || !Yout || !Zout) return set_err(ctx, SPAMM_EINVAL, "NULL argument");
    if (iters < 1) return set_err(ctx, SPAMM_EINVAL, "iters must be >= 1");
    if (!(tau >= 0.0) || !std::isfinite(tau)) return set_err(ctx, SPAMM_EINVAL, "tau must be finite and >= 0");
    if (s->dist) return set_err(ctx, SPAMM_EINVAL, "single channel needs Z^T: not on a row-partitioned context");
    spamm_ns_opts o{};
    o.tau_s = -1.0;
    o.power_iters = 100;
    if (opts) o = *opts;
    if (o.power_iters <= 0) o.power_iters = 100;
    if (o.mu != 0.0) return set_err(ctx, SPAMM_EINVAL, "mu is not supported by the single channel");
    const double tau_s = o.tau_s < 0.0 ? tau : o.tau_s;
    int ps = prof_begin(ctx, SPAMM_PH_SETUP);
    double root = 0.0;
    ST(spamm_norm(ctx, s, &root));
    if (!(root > 0.0)) return set_err(ctx, SPAMM_EINVAL, "s is zero");
    double c = o.scale;
    if (!(c > 0.0)) ST(power_scale(ctx, s, o.power_iters, &c));
    if (o.c_out) *o.c_out = c;
    if (o.iters_done) *o.iters_done = 0;
    spamm_mat S1 = nullptr, Z = nullptr, H = nullptr, W = nullptr;
    ST(spamm_ns_y0(ctx, s, c, 0.0, &S1));                 // s' = s/c = X_0
    spamm_status st = spamm_identity(ctx, s->n, s->b, &Z);
    if (!st) st = h_of(ctx, S1, o.map, &H);                // H_0 = h[X_0], t_0 -> dscratch
    double t = 0.0;
    if (!st) {
        ST(fetch1(ctx, ctx->dscratch, &t, sizeof(double)));
    }
    if (!st) st = mat_map(ctx, S1, 2, 1.0, 0.0, &W);       // W_0 = s' (replaced by the first step)
    prof_end(ctx, ps);
    int pl = prof_begin(ctx, SPAMM_PH_LOOP);
    for (int k = 0; k < iters && !st; k++) {
        if (o.t_history) o.t_history[k] = t;
        spamm_mat Zn = nullptr, Hn = nullptr, Wn = nullptr;
        double tn = 0.0;
        spamm_stats sts[3];
        st = spamm_ns_step_single(ctx, S1, Z, H, tau, tau_s, o.map, &Zn, &Hn, &Wn, &tn, sts, nullptr);
        if (o.per_product && st == SPAMM_OK) memcpy(o.per_product + 3 * k, sts, sizeof(sts));
        if (st) {
            spamm_mat_free(Zn);
            spamm_mat_free(Hn);
            spamm_mat_free(Wn);
            break;
        }
        spamm_mat_free(Z);
        spamm_mat_free(H);
        spamm_mat_free(W);
        Z = Zn;
        H = Hn;
        W = Wn;
        if (o.iters_done) *o.iters_done = k + 1;
        const double tk = t;
        t = tn;
        if (o.t_stop > 0.0 && std::fabs(tk) <= o.t_stop) break;
    }
    prof_end(ctx, pl);
    std::string err = ctx->err;
    spamm_status st2 = SPAMM_OK;
    if (Z && W) {
        const double f = std::sqrt(c);
        spamm_mat Yf = nullptr, Zf = nullptr;
        st2 = mat_map(ctx, W, 2, f, 0.0, &Yf);
        if (!st2) st2 = mat_map(ctx, Z, 0, f, 0.0, &Zf);
        if (!st2) {
            *Yout = Yf;
            *Zout = Zf;
        } else {
            spamm_mat_free(Yf);
            spamm_mat_free(Zf);
        }
    }
    spamm_mat_free(S1);
    spamm_mat_free(Z);
    spamm_mat_free(H);
    spamm_mat_free(W);
    if (st) {
        ctx->err = err;
        return st;
    }
    return st2;
}

// ------------------------------------- regularised product representation
// Eq. product_rep (reading L21), SURVEY.md §8(f) f3:
//   c = ||s||_2, S_i = s/c + mu_i I, R_0 = S_0, R_i = F^T (x)_tau1 (S_i (x)_tau1 F),
//   Z_i = R_i^{-1/2} (dual iteration at tau = tau_s = tau0), F = Z_0, F <- F (x)_tau1 Z_i;
//   G = F / sqrt(c) with G^T (s + c mu_m I) G ~ I.  Single device (uses F^T).
extern "C" spamm_status spamm_regularized_factor(spamm_ctx ctx, spamm_mat s, double tau0, double tau1,
                                                 const double *mu, int32_t nslices, int32_t iters, double t_stop,
                                                 double scale, spamm_mat *G, double *c_out, int32_t *slice_iters)
{
    if (!ctx || !s || !mu || !G || nslices < 1 || iters < 1) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    if (!(tau0 >= 0.0) || !(tau1 >= 0.0)) return set_err(ctx, SPAMM_EINVAL, "tau must be >= 0");
    if (s->dist) return set_err(ctx, SPAMM_EINVAL, "regularised slices need F^T: not on a row-partitioned context");
    double c = scale;
    if (!(c > 0.0)) ST(power_scale(ctx, s, 100, &c));
    if (c_out) *c_out = c;
    spamm_mat F = nullptr;
    spamm_status st = SPAMM_OK;
    for (int i = 0; i < nslices && !st; i++) {
        spamm_mat Si = nullptr, R = nullptr;
        st = mat_map(ctx, s, 8, c, mu[i], &Si);
        if (st) break;
        if (!F) {
            R = Si;
        } else {
            spamm_mat W = nullptr;
            st = product(ctx, ctx->cw[0], Si, F, tau1, EPI_STORE, nullptr, &W);
            if (!st) st = product(ctx, ctx->cw[1], F, W, tau1, EPI_STORE, nullptr, &R, 1);
            spamm_mat_free(W);
            spamm_mat_free(Si);
            if (st) break;
        }
        spamm_ns_opts o{};
        o.tau_s = tau0;
        o.power_iters = 100;
        o.t_stop = t_stop;
        int32_t done = 0;
        o.iters_done = &done;
        spamm_mat Y = nullptr, Z = nullptr;
        st = spamm_ns_sqrt(ctx, R, tau0, iters, &Y, &Z, &o);
        if (slice_iters) slice_iters[i] = done;
        spamm_mat_free(R);
        spamm_mat_free(Y);
        if (st) {
            spamm_mat_free(Z);
            break;
        }
        if (!F) {
            F = Z;
        } else {
            spamm_mat Fn = nullptr;
            st = product(ctx, ctx->cw[2], F, Z, tau1, EPI_STORE, nullptr, &Fn);
            spamm_mat_free(Z);
            if (!st) {
                spamm_mat_free(F);
                F = Fn;
            }
        }
    }
    if (!st) st = mat_map(ctx, F, 0, std::sqrt(c), 0.0, G);
    spamm_mat_free(F);
    return st;
}
