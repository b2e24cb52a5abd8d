// prof.cu — measurement utilities: phase timing with CUDA events on the context
// stream (roofline of the dominant kernel in bench.py), the FP64 DMMA issue-rate
// peak microbenchmark, and block export.
#include <vector>

#include "common.cuh"

struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t next = 0;
    struct Iv {
        int phase;
        cudaEvent_t a, b;
    };
    std::vector<Iv> ivs;
    double gemm_flops = 0, gemm_bytes = 0;
    int64_t gemm_tasks = 0;
};

static Prof *prof_of(spamm_ctx ctx)
{
    if (!ctx->prof) ctx->prof = new Prof();
    return (Prof *)ctx->prof;
}

static cudaEvent_t ev_get(Prof *p)
{
    if (p->next == p->pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        p->pool.push_back(e);
    }
    return p->pool[p->next++];
}

int prof_begin(spamm_ctx ctx, int phase)
{
    Prof *p = (Prof *)ctx->prof;
    if (!p || !p->on || ctx->capturing) return -1;
    cudaEvent_t a = ev_get(p);
    cudaEventRecord(a, ctx->stream);
    p->ivs.push_back({phase, a, nullptr});
    return (int)p->ivs.size() - 1;
}

void prof_end(spamm_ctx ctx, int idx)
{
    if (idx < 0) return;
    Prof *p = (Prof *)ctx->prof;
    cudaEvent_t b = ev_get(p);
    cudaEventRecord(b, ctx->stream);
    p->ivs[idx].b = b;
}

void prof_gemm_work(spamm_ctx ctx, int64_t tasks, int64_t segs, int b)
{
    Prof *p = (Prof *)ctx->prof;
    if (!p || !p->on) return;
    double b2 = (double)b * b;
    p->gemm_tasks += tasks;
    p->gemm_flops += 2.0 * b2 * b * (double)tasks;
    p->gemm_bytes += 8.0 * b2 * (2.0 * (double)tasks + (double)segs);
}

void prof_destroy(spamm_ctx ctx)
{
    Prof *p = (Prof *)ctx->prof;
    if (!p) return;
    for (auto e : p->pool) cudaEventDestroy(e);
    delete p;
    ctx->prof = nullptr;
}

extern "C" spamm_status spamm_profile_enable(spamm_ctx ctx, int32_t enable)
{
    if (!ctx) return SPAMM_EINVAL;
    Prof *p = prof_of(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    p->on = enable != 0;
    p->ivs.clear();
    p->next = 0;
    p->gemm_flops = p->gemm_bytes = 0;
    p->gemm_tasks = 0;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_profile_read(spamm_ctx ctx, spamm_profile_t *out)
{
    if (!ctx || !out) return SPAMM_EINVAL;
    Prof *p = prof_of(ctx);
    CK(cudaStreamSynchronize(ctx->stream));
    *out = spamm_profile_t{};
    for (auto &iv : p->ivs) {
        if (!iv.b) continue;
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, iv.a, iv.b));
        out->ms[iv.phase] += ms;
        out->count[iv.phase]++;
    }
    out->gemm_flops = p->gemm_flops;
    out->gemm_tasks = p->gemm_tasks;
    out->gemm_operand_bytes = p->gemm_bytes;
    return SPAMM_OK;
}

// ----------------------------------------------------------- DMMA peak
__global__ void __launch_bounds__(256) k_peak_dmma(const double *seed, int64_t iters, double *out)
{
    double a = seed[threadIdx.x & 31], b = seed[32 + (threadIdx.x & 31)];
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
    for (int64_t it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;  // keep the work observable
}

extern "C" spamm_status spamm_peak_dmma(spamm_ctx ctx, int64_t iters, double *tflops, double *ms_out)
{
    if (!ctx || !tflops) return SPAMM_EINVAL;
    double *seed = dalloc<double>(ctx, 64);
    CK(cudaMemsetAsync(seed, 0, sizeof(double) * 64, ctx->stream));
    const int ctas = ctx->sm_count * 4, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_peak_dmma<<<ctas, threads, 0, ctx->stream>>>(seed, iters / 10 + 1, seed + 48);  // warm-up
    cudaEventRecord(a, ctx->stream);
    k_peak_dmma<<<ctas, threads, 0, ctx->stream>>>(seed, iters, seed + 48);
    cudaEventRecord(b, ctx->stream);
    CKL(ctx);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    dev_free(ctx, seed, sizeof(double) * 64);
    double flops = (double)ctas * (threads / 32) * (double)iters * 8.0 * 512.0;
    *tflops = flops / (ms * 1e-3) / 1e12;
    if (ms_out) *ms_out = ms;
    return SPAMM_OK;
}

// ------------------------------------------------------------ export
__global__ void k_coords_out(const int32_t *coord, int64_t n, int32_t *bi, int32_t *bj)
{
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint32_t c = coord[t];
    bi[t] = morton_i(c);
    bj[t] = morton_j(c);
}

__global__ void k_unswizzle(const double *pool, int b, double *out)
{
    const int64_t blk = blockIdx.x;
    const double *s = pool + blk * (int64_t)b * b;
    double *d = out + blk * (int64_t)b * b;
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) d[e] = s[pool_at(e / b, e % b, b)];
}

extern "C" spamm_status spamm_export_blocks(spamm_ctx ctx, spamm_mat m, int32_t *bi, int32_t *bj,
                                            double *blocks, int64_t cap, int64_t *n)
{
    if (!ctx || !m || !n) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    *n = m->nblk;
    int64_t k = m->nblk < cap ? m->nblk : cap;
    if (k <= 0) return SPAMM_OK;
    if (!bi || !bj || !blocks) return set_err(ctx, SPAMM_EINVAL, "NULL output");
    const int64_t b2 = (int64_t)m->b * m->b;
    bool hc = !is_device_ptr(bi), hb = !is_device_ptr(blocks);
    int32_t *dbi = hc ? dalloc<int32_t>(ctx, k) : bi, *dbj = hc ? dalloc<int32_t>(ctx, k) : bj;
    k_coords_out<<<cdiv(k, 256), 256, 0, ctx->stream>>>(m->coord, k, dbi, dbj);
    CKL(ctx);
    if (hc) {
        CK(cudaMemcpyAsync(bi, dbi, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(bj, dbj, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, ctx->stream));
    }
    // un-swizzle into row-major blocks (device), then one copy out if the target is host
    double *dbl = hb ? dalloc<double>(ctx, k * b2) : blocks;
    if (!dbl) return set_err(ctx, SPAMM_ENOMEM, "export staging");
    k_unswizzle<<<(int)k, 256, 0, ctx->stream>>>(m->pool, m->b, dbl);
    CKL(ctx);
    if (hb) CK(cudaMemcpyAsync(blocks, dbl, sizeof(double) * k * b2, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (hb) dev_free(ctx, dbl, sizeof(double) * k * b2);
    if (hc) {
        dev_free(ctx, dbi, sizeof(int32_t) * k);
        dev_free(ctx, dbj, sizeof(int32_t) * k);
    }
    return SPAMM_OK;
}

