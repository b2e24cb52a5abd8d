// hostio.cu — asynchronous host I/O of the C ABI: uploads of block-list inputs on the
// library's upload stream (spamm_stage_blocks -> spamm_build_tree_staged) and exports of
// results on its copy stream (spamm_export_blocks_async), so a caller can keep the
// device busy while the previous result and the next input cross PCIe.  Staging lives
// in context-owned slots reused round-robin, each guarded by CUDA events (never freed
// while a copy may still touch it).
#include <algorithm>

#include "common.cuh"

__global__ void k_coords_out(const int32_t *coord, int64_t n, int32_t *bi, int32_t *bj);
__global__ void k_unswizzle(const double *pool, int b, double *out);

// ------------------------------------------------------- asynchronous export
// Staging slots owned by the context: the un-swizzle runs on the context stream into
// slot q, the device->host copy on the context's copy stream (a separate copy engine
// queue) after an event, so it overlaps the context stream's next work.  A slot is
// reused only after its previous copy's event (the context stream waits on it).
struct XSlot {
    void *dev = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;
};
struct ISlot {
    void *dev = nullptr;
    size_t bytes = 0;
    cudaEvent_t loaded = nullptr, consumed = nullptr;
    int64_t gen = 0;
};
struct XState {
    cudaStream_t copy = nullptr;
    cudaEvent_t ready = nullptr, last = nullptr;
    XSlot slot[SPAMM_XSLOTS];
    int next = 0;
    // uploads
    cudaStream_t up = nullptr;
    ISlot in[SPAMM_ISLOTS];
    int in_next = 0;
};

static spamm_status xstate(spamm_ctx ctx, XState **out)
{
    if (!ctx->xs) {
        XState *x = new XState();
        ctx->xs = x;
        CK(cudaStreamCreateWithFlags(&x->copy, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&x->ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&x->last, cudaEventDisableTiming));
        for (auto &q : x->slot) CK(cudaEventCreateWithFlags(&q.done, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&x->up, cudaStreamNonBlocking));
        for (auto &q : x->in) {
            CK(cudaEventCreateWithFlags(&q.loaded, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&q.consumed, cudaEventDisableTiming));
        }
    }
    *out = (XState *)ctx->xs;
    return SPAMM_OK;
}

void xstate_free(spamm_ctx ctx)
{
    XState *x = (XState *)ctx->xs;
    if (!x) return;
    if (x->copy) cudaStreamSynchronize(x->copy);
    if (x->up) cudaStreamSynchronize(x->up);
    for (auto &q : x->in) {
        dev_free(ctx, q.dev, q.bytes);
        if (q.loaded) cudaEventDestroy(q.loaded);
        if (q.consumed) cudaEventDestroy(q.consumed);
    }
    if (x->up) cudaStreamDestroy(x->up);
    for (auto &q : x->slot) {
        dev_free(ctx, q.dev, q.bytes);
        if (q.done) cudaEventDestroy(q.done);
    }
    if (x->ready) cudaEventDestroy(x->ready);
    if (x->last) cudaEventDestroy(x->last);
    if (x->copy) cudaStreamDestroy(x->copy);
    delete x;
    ctx->xs = nullptr;
}

extern "C" spamm_status spamm_export_blocks_async(spamm_ctx ctx, spamm_mat m, int32_t *bi, int32_t *bj,
                                                  double *blocks, int64_t cap, int64_t *n)
{
    if (!ctx || !m || !n) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    *n = m->nblk;
    const int64_t k = m->nblk < cap ? m->nblk : cap;
    if (k <= 0) return SPAMM_OK;
    if (!bi || !bj || !blocks) return set_err(ctx, SPAMM_EINVAL, "NULL output");
    if (is_device_ptr(bi) || is_device_ptr(bj) || is_device_ptr(blocks))
        return set_err(ctx, SPAMM_EINVAL, "spamm_export_blocks_async writes host buffers");
    XState *x = nullptr;
    ST(xstate(ctx, &x));
    XSlot &q = x->slot[x->next];
    x->next = (x->next + 1) % SPAMM_XSLOTS;
    const int64_t b2 = (int64_t)m->b * m->b;
    const size_t need = sizeof(double) * k * b2 + 2 * sizeof(int32_t) * k + 512;
    CK(cudaStreamWaitEvent(ctx->stream, q.done, 0));   // the slot's previous copy is over
    if (q.bytes < need) {
        dev_free(ctx, q.dev, q.bytes);
        q.bytes = need + need / 4;
        q.dev = dev_alloc(ctx, q.bytes);
        if (!q.dev) {
            q.bytes = 0;
            return set_err(ctx, SPAMM_ENOMEM, "export staging (%lld blocks)", (long long)k);
        }
    }
    double *dbl = (double *)q.dev;
    int32_t *dbi = (int32_t *)(dbl + k * b2), *dbj = dbi + k;
    k_coords_out<<<cdiv(k, 256), 256, 0, ctx->stream>>>(m->coord, k, dbi, dbj);
    CKL(ctx);
    k_unswizzle<<<(int)k, 256, 0, ctx->stream>>>(m->pool, m->b, dbl);
    CKL(ctx);
    CK(cudaEventRecord(x->ready, ctx->stream));
    CK(cudaStreamWaitEvent(x->copy, x->ready, 0));
    CK(cudaMemcpyAsync(blocks, dbl, sizeof(double) * k * b2, cudaMemcpyDeviceToHost, x->copy));
    CK(cudaMemcpyAsync(bi, dbi, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, x->copy));
    CK(cudaMemcpyAsync(bj, dbj, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, x->copy));
    CK(cudaEventRecord(q.done, x->copy));
    CK(cudaEventRecord(x->last, x->copy));
    return SPAMM_OK;
}

extern "C" spamm_status spamm_copies_join(spamm_ctx ctx)
{
    if (!ctx) return SPAMM_EINVAL;
    if (!ctx->xs) return SPAMM_OK;
    CK(cudaStreamWaitEvent(ctx->stream, ((XState *)ctx->xs)->last, 0));
    return SPAMM_OK;
}

extern "C" spamm_status spamm_copies_wait(spamm_ctx ctx)
{
    if (!ctx) return SPAMM_EINVAL;
    if (!ctx->xs) return SPAMM_OK;
    CK(cudaEventSynchronize(((XState *)ctx->xs)->last));
    return SPAMM_OK;
}

// ------------------------------------------------------------------ uploads
struct spamm_staged_s {
    int slot;
    int64_t gen, nblocks;   // block list: nblocks; dense: -1
    int b;
    int64_t n;              // dense: n x n, row-major (ld = n in the slot)
};

// slot qi refilled with `bytes` from the upload stream (grown when needed)
static spamm_status slot_fill(spamm_ctx ctx, XState *x, int qi, size_t need)
{
    ISlot &q = x->in[qi];
    if (q.bytes < need) {
        // growth (rare): the slot's previous upload and build must be over first
        CK(cudaEventSynchronize(q.loaded));
        CK(cudaEventSynchronize(q.consumed));
        dev_free(ctx, q.dev, q.bytes);
        q.bytes = need + need / 8;
        q.dev = dev_alloc(ctx, q.bytes);
        if (!q.dev) {
            q.bytes = 0;
            return set_err(ctx, SPAMM_ENOMEM, "upload staging (%lld bytes)", (long long)need);
        }
        CK(cudaStreamSynchronize(ctx->stream));   // the allocation is usable on any stream
    }
    CK(cudaStreamWaitEvent(x->up, q.consumed, 0));   // the slot's previous build has read it
    return SPAMM_OK;
}

extern "C" spamm_status spamm_stage_blocks(spamm_ctx ctx, int64_t nblocks, int32_t b, const int32_t *bi,
                                           const int32_t *bj, const double *blocks, spamm_staged *out)
{
    if (!ctx || !out || nblocks < 0 || (nblocks > 0 && (!bi || !bj || !blocks)))
        return set_err(ctx, SPAMM_EINVAL, "bad argument");
    *out = nullptr;
    if (b != 16 && b != 32 && b != 64) return set_err(ctx, SPAMM_EINVAL, "b=%d not in {16,32,64}", b);
    if (is_device_ptr(bi) || is_device_ptr(bj) || is_device_ptr(blocks))
        return set_err(ctx, SPAMM_EINVAL, "spamm_stage_blocks reads host buffers");
    XState *x = nullptr;
    ST(xstate(ctx, &x));
    const int qi = x->in_next;
    ISlot &q = x->in[qi];
    x->in_next = (x->in_next + 1) % SPAMM_ISLOTS;
    const int64_t b2 = (int64_t)b * b;
    ST(slot_fill(ctx, x, qi, sizeof(double) * nblocks * b2 + 2 * sizeof(int32_t) * nblocks + 1024));
    double *dbl = (double *)q.dev;
    int32_t *dbi = (int32_t *)(dbl + nblocks * b2), *dbj = dbi + nblocks;
    if (nblocks > 0) {
        CK(cudaMemcpyAsync(dbl, blocks, sizeof(double) * nblocks * b2, cudaMemcpyHostToDevice, x->up));
        CK(cudaMemcpyAsync(dbi, bi, sizeof(int32_t) * nblocks, cudaMemcpyHostToDevice, x->up));
        CK(cudaMemcpyAsync(dbj, bj, sizeof(int32_t) * nblocks, cudaMemcpyHostToDevice, x->up));
    }
    CK(cudaEventRecord(q.loaded, x->up));
    q.gen++;
    *out = new spamm_staged_s{qi, q.gen, nblocks, b, 0};
    return SPAMM_OK;
}

extern "C" spamm_status spamm_stage_dense(spamm_ctx ctx, const double *dense, int64_t n, int64_t ld,
                                          spamm_staged *out)
{
    if (!ctx || !out || !dense || n <= 0 || ld < n) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    *out = nullptr;
    if (is_device_ptr(dense)) return set_err(ctx, SPAMM_EINVAL, "spamm_stage_dense reads host memory");
    XState *x = nullptr;
    ST(xstate(ctx, &x));
    const int qi = x->in_next;
    ISlot &q = x->in[qi];
    x->in_next = (x->in_next + 1) % SPAMM_ISLOTS;
    ST(slot_fill(ctx, x, qi, sizeof(double) * n * n + 1024));
    CK(cudaMemcpy2DAsync(q.dev, sizeof(double) * n, dense, sizeof(double) * ld, sizeof(double) * n, n,
                         cudaMemcpyHostToDevice, x->up));
    CK(cudaEventRecord(q.loaded, x->up));
    q.gen++;
    *out = new spamm_staged_s{qi, q.gen, -1, 0, n};
    return SPAMM_OK;
}

extern "C" spamm_status spamm_build_tree_staged(spamm_ctx ctx, int64_t n, int32_t b, spamm_staged staged,
                                                spamm_mat *out)
{
    if (!ctx || !staged || !out) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    XState *x = (XState *)ctx->xs;
    ISlot &q = x->in[staged->slot];
    if (q.gen != staged->gen) {
        delete staged;
        return set_err(ctx, SPAMM_EINVAL, "staged upload overwritten (more than %d uploads outstanding)",
                       SPAMM_ISLOTS);
    }
    spamm_status st = SPAMM_OK;
    if (staged->nblocks >= 0 && staged->b != b) st = set_err(ctx, SPAMM_EINVAL, "b differs from the upload's");
    if (staged->nblocks < 0 && staged->n != n) st = set_err(ctx, SPAMM_ESHAPE, "n differs from the upload's");
    if (!st && cudaStreamWaitEvent(ctx->stream, q.loaded, 0) != cudaSuccess)
        st = set_err(ctx, SPAMM_ECUDA, "upload wait");
    if (!st && staged->nblocks < 0) {
        st = spamm_build_tree(ctx, (const double *)q.dev, n, n, b, out);
    } else if (!st) {
        const int64_t nbk = staged->nblocks, b2 = (int64_t)b * b;
        const double *dbl = (const double *)q.dev;
        const int32_t *dbi = (const int32_t *)(dbl + nbk * b2), *dbj = dbi + nbk;
        st = spamm_build_tree_blocks(ctx, n, b, nbk, dbi, dbj, dbl, out);
    }
    cudaEventRecord(q.consumed, ctx->stream);   // the slot may be refilled after the build
    delete staged;
    return st;
}

extern "C" void spamm_staged_free(spamm_staged staged) { delete staged; }
