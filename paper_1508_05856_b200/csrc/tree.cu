// tree.cu — quadtree construction and maintenance on the device.
//
// the quadtree matrix a^i with children a^{i+1}_{xy} and the
// Frobenius recursion ||a^i|| = sqrt(sum ||a^{i+1}_xy||^2).  Here the norms are
// stored squared (reading L5) in a Morton-ordered pyramid so that the four
// children of a node are one 32-byte sector, and the leaves live in a packed,
// slot-indexed block pool.  Kernels:
//   k_block_norm2     one warp per candidate block, coalesced double2 loads,
//                     fixed-order shuffle tree (deterministic)        [HBM-bound]
//   k_build_scatter   order-preserving compaction of present blocks (scan.cuh)
//   k_pyramid         CTA-local reduction of 5 levels per launch       [L2-bound]
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "common.cuh"
#include "scan.cuh"

// ---------------------------------------------------------------- errors
spamm_status set_err(spamm_ctx ctx, spamm_status st, const char *fmt, ...)
{
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        ctx->err = buf;
    }
    return st;
}

spamm_status check_cuda(spamm_ctx ctx, cudaError_t e, const char *what)
{
    return set_err(ctx, e == cudaErrorMemoryAllocation ? SPAMM_ENOMEM : SPAMM_ECUDA,
                   "CUDA error %s (%d) in %s", cudaGetErrorString(e), (int)e, what);
}

// ---------------------------------------------------------------- memory
// SPAMM_POISON=1 (debug): every allocation is filled with 0xFF bytes (NaN doubles,
// -1 ints) so a read of memory no kernel wrote shows up as NaN / a bad slot.
static int poison_mode()
{
    static const int m = [] {   // initialised once, thread-safely (C++11)
        const char *e = getenv("SPAMM_POISON");
        return (e && *e == '1') ? 1 : 0;
    }();
    return m;
}

// The context's own pool (no allocator given): requests of 32 MiB and more are rounded up
// to 4 size classes per octave (<= 25 % slack).  The NS iterates grow a little every step
// (fill-in), so an exact-size request never fits a freed block and the pool would map new
// memory for every product (C3: 335 vs 232 ms per run); with classes, freed iterates serve
// the next step's requests.
static size_t pool_class(size_t bytes)
{
    if (bytes < ((size_t)32 << 20)) return bytes;
    int e = 63 - __builtin_clzll((unsigned long long)bytes);
    const size_t q = (size_t)1 << (e - 2);
    return (bytes + q - 1) & ~(q - 1);
}

void *dev_alloc(spamm_ctx ctx, size_t bytes)
{
    bytes = (bytes + 255) & ~size_t(255);
    void *p = nullptr;
    if (!ctx->has_alloc) bytes = pool_class(bytes);
    if (ctx->has_alloc) {
        p = ctx->alloc.alloc(bytes, (void *)ctx->stream, ctx->alloc.user);
    } else if ((ctx->pool ? cudaMallocFromPoolAsync(&p, bytes, ctx->pool, ctx->stream)
                          : cudaMallocAsync(&p, bytes, ctx->stream)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (p && poison_mode()) cudaMemsetAsync(p, 0xFF, bytes, ctx->stream);
    return p;
}

void dev_free(spamm_ctx ctx, void *p, size_t bytes)
{
    if (!p) return;
    bytes = (bytes + 255) & ~size_t(255);
    if (ctx->has_alloc) ctx->alloc.free(p, bytes, (void *)ctx->stream, ctx->alloc.user);
    else cudaFreeAsync(p, ctx->stream);
}

struct FetchArgs {
    const uint32_t *src[8];
    uint32_t words[8];
    uint32_t off[8];
    int n;
};

__global__ void k_fetch(FetchArgs a, uint32_t *dst)
{
    for (int i = 0; i < a.n; i++)
        for (uint32_t w = threadIdx.x; w < a.words[i]; w += blockDim.x) dst[a.off[i] + w] = a.src[i][w];
}

spamm_status fetch(spamm_ctx ctx, const FetchItem *items, int n)
{
    if (!ctx->zc) {
        CK(cudaHostAlloc(&ctx->zc, SPAMM_ZC_BYTES, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(&ctx->zc_dev, ctx->zc, 0));
    }
    for (int i0 = 0; i0 < n; i0 += 8) {
        FetchArgs a{};
        uint32_t off = 0;
        for (int i = i0; i < n && i < i0 + 8; i++) {
            if (items[i].bytes % 4 || off * 4 + items[i].bytes > SPAMM_ZC_BYTES)
                return set_err(ctx, SPAMM_EINVAL, "fetch of %u bytes", items[i].bytes);
            a.src[a.n] = (const uint32_t *)items[i].src;
            a.words[a.n] = items[i].bytes / 4;
            a.off[a.n] = off;
            off += items[i].bytes / 4;
            a.n++;
        }
        k_fetch<<<1, 256, 0, ctx->stream>>>(a, (uint32_t *)ctx->zc_dev);
        CKL(ctx);
        CK(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < a.n; i++) memcpy(items[i0 + i].dst, (const uint32_t *)ctx->zc + a.off[i], items[i0 + i].bytes);
    }
    return SPAMM_OK;
}

int is_device_ptr(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

spamm_status mat_new(spamm_ctx ctx, int64_t n, int b, int64_t cap, spamm_mat *out)
{
    if (b != 16 && b != 32 && b != 64)
        return set_err(ctx, SPAMM_EINVAL, "leaf size b=%d not in {16,32,64}", b);
    if (n < b || n % b) return set_err(ctx, SPAMM_EINVAL, "n=%lld not a multiple of b", (long long)n);
    int64_t nb = n / b;
    if (nb & (nb - 1)) return set_err(ctx, SPAMM_EINVAL, "n/b=%lld not a power of two", (long long)nb);
    int L = 0;
    while ((int64_t(1) << L) < nb) L++;
    if (L > SPAMM_MAX_L) return set_err(ctx, SPAMM_EINVAL, "n/b too large");
    Parts parts;
    ST(mat_parts(ctx, (int)nb, &parts));
    spamm_mat m = new spamm_mat_s();
    m->ctx = ctx;
    ctx->live_mats.fetch_add(1);
    m->n = n; m->b = b; m->nb = (int)nb; m->L = L;
    m->cap = cap;
    m->parts = parts;
    m->dist = ctx->comm != nullptr;
    m->r0 = m->dist ? parts.rs[ctx->comm->rank] : 0;
    m->r1 = m->dist ? parts.rs[ctx->comm->rank + 1] : (int)nb;
    m->norm2 = dalloc<double>(ctx, pyr_size(L));
    m->slot = dalloc<int32_t>(ctx, nb * nb);
    m->pool = dalloc<double>(ctx, cap * b * b);
    m->coord = dalloc<int32_t>(ctx, cap);
    if (!m->norm2 || !m->slot || !m->pool || !m->coord) {
        spamm_mat_free(m);
        return set_err(ctx, SPAMM_ENOMEM, "allocation of a %lld-block matrix failed", (long long)cap);
    }
    *out = m;
    return SPAMM_OK;
}

extern "C" void spamm_mat_free(spamm_mat m)
{
    if (!m) return;
    spamm_ctx ctx = m->ctx;
    int64_t nb = m->nb;
    dev_free(ctx, m->norm2, sizeof(double) * pyr_size(m->L));
    dev_free(ctx, m->slot, sizeof(int32_t) * nb * nb);
    dev_free(ctx, m->pool, sizeof(double) * (size_t)(m->cap > 0 ? m->cap : 1) * m->b * m->b);
    dev_free(ctx, m->coord, sizeof(int32_t) * (m->cap > 0 ? m->cap : 1));
    delete m;
    // the last matrix of a context whose destroy was deferred
    if (ctx->live_mats.fetch_sub(1) == 1 && ctx->destroy_pending.load()) ctx_teardown(ctx);
}

spamm_status mat_reset_pattern(spamm_ctx ctx, spamm_mat m)
{
    CK(cudaMemsetAsync(m->slot, 0xFF, sizeof(int32_t) * (size_t)m->nb * m->nb, ctx->stream));
    CK(cudaMemsetAsync(m->norm2, 0, sizeof(double) * pyr_size(m->L), ctx->stream));
    return SPAMM_OK;
}

// ---------------------------------------------------------------- kernels
// Sum of squares of a b*b block (row-major, row stride ld doubles), one warp,
// fixed order: lane-strided double2 partials then an xor-shuffle tree.
__device__ __forceinline__ double warp_block_sumsq(const double *blk, int b, int64_t ld, int lane)
{
    double s0 = 0.0, s1 = 0.0;
    const int half = b / 2;  // double2 per row
#pragma unroll 8
    for (int q = lane; q < b * half; q += 32) {
        int r = q / half, c = (q % half) * 2;
        double2 v = *reinterpret_cast<const double2 *>(blk + (int64_t)r * ld + c);
        s0 = fma(v.x, v.x, s0);
        s1 = fma(v.y, v.y, s1);
    }
    double s = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// Block source: a block list (bi, bj, blocks) or a dense matrix (implicit (I,J)).
struct BlockSrc {
    const int32_t *bi, *bj;
    const double *blocks;  // list mode
    const double *dense;   // dense mode
    int64_t ld;
    int b, nb;
    __device__ __forceinline__ void coords(int64_t t, int &I, int &J) const
    {
        if (dense) { I = (int)(t / nb); J = (int)(t % nb); }
        else { I = bi[t]; J = bj[t]; }
    }
    __device__ __forceinline__ const double *ptr(int64_t t, int64_t &stride) const
    {
        if (dense) {
            int I = (int)(t / nb), J = (int)(t % nb);
            stride = ld;
            return dense + (int64_t)I * b * ld + (int64_t)J * b;
        }
        stride = b;
        return blocks + t * (int64_t)b * b;
    }
};

__global__ void k_block_norm2(BlockSrc src, int64_t count, double *n2)
{
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (w >= count) return;
    int64_t ld;
    const double *p = src.ptr(w, ld);
    double s = warp_block_sumsq(p, src.b, ld, lane);
    if (lane == 0) n2[w] = s;
}

// Order-preserving compaction of present blocks (n2 > 0): exclusive scan of the
// present flags gives the pool slot; the block is copied and registered.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_build_scan(BlockSrc src, const double *n2, int64_t count,
                                                        int r0, int r1, ScanTiles<V1> st, int32_t *slot_of)
{
    __shared__ V1 sw[THREADS / 32];
    __shared__ int s_tile, s_excl;
    int tile;
    while ((tile = next_tile(st.ticket, count, THREADS, &s_tile)) >= 0) {
        int64_t t = (int64_t)tile * THREADS + threadIdx.x;
        int I = 0, J = 0;
        if (t < count) src.coords(t, I, J);
        // present (reading L6) and in the local block rows (row partition, §8(e))
        V1 v{(t < count && n2[t] > 0.0 && I >= r0 && I < r1) ? 1 : 0};
        V1 tot;
        V1 ex = block_excl_scan<V1, THREADS>(v, &tot, sw);
        if (threadIdx.x < 32) {
            int e = tile_lookback(st, tile, tot).x;
            if (threadIdx.x == 0) s_excl = e;
        }
        __syncthreads();
        if (t < count) slot_of[t] = v.x ? s_excl + ex.x : -1;
        __syncthreads();
    }
}

__global__ void k_build_scatter(BlockSrc src, int64_t count, const int32_t *slot_of,
                                const double *n2, int L, double *pool, int32_t *coord,
                                int32_t *slot_map, double *leaf_n2)
{
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (w >= count) return;
    int s = slot_of[w];
    if (s < 0) return;
    int I, J;
    src.coords(w, I, J);
    uint32_t code = morton(I, J);
    int64_t ld;
    const double *p = src.ptr(w, ld);
    const int b = src.b, half = b / 2;
    double *dst = pool + (int64_t)s * b * b;
    for (int q = lane; q < b * half; q += 32) {
        int r = q / half, c = (q % half) * 2;
        *reinterpret_cast<double2 *>(dst + pool_at(r, c, b)) =
            *reinterpret_cast<const double2 *>(p + (int64_t)r * ld + c);
    }
    if (lane == 0) {
        coord[s] = (int32_t)code;
        slot_map[code] = s;
        leaf_n2[code] = n2[w];
    }
}

// Pyramid: each CTA reduces 4^LV consecutive entries of level `lf` into levels
// lf-1 .. lf-LV (fixed order (c0+c1)+(c2+c3)).
// tail > 0: the last CTA to finish (a counter in the root level's padding, norm2[1..3],
// which is zero between uses) also forms the `tail` levels above lf - levels from the
// values the other CTAs stored -- one launch instead of two, the same (c0 + c1) + (c2 + c3)
// per node, so the same bits.
template <int LV>
__global__ void k_pyramid(double *norm2, int lf, int levels, int tail, double *norm2b, int grida)
{
    pdl_wait();
    pdl_trigger();
    // norm2b (nullable): a second pyramid of the same shape built by CTAs grida.. of the same
    // launch (the Y' and Z' pyramids of a captured NS step)
    const bool second = norm2b && (int)blockIdx.x >= grida;
    if (second) norm2 = norm2b;
    const int bid = second ? blockIdx.x - grida : blockIdx.x;
    const int ncta = norm2b ? (second ? gridDim.x - grida : grida) : gridDim.x;
    constexpr int N = 1 << (2 * LV);
    __shared__ double buf[N];
    const int64_t base = (int64_t)bid * N;
    const double *src = norm2 + pyr_off(lf);
    const int64_t cnt = int64_t(1) << (2 * lf);
    for (int i = threadIdx.x; i < N; i += blockDim.x) buf[i] = (base + i < cnt) ? src[base + i] : 0.0;
    __syncthreads();
    int m = N;
    for (int k = 1; k <= levels; k++) {
        m >>= 2;
        double *dst = norm2 + pyr_off(lf - k);
        double v[8];
        int nloc = 0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            double c0 = buf[4 * i], c1 = buf[4 * i + 1], c2 = buf[4 * i + 2], c3 = buf[4 * i + 3];
            v[nloc++] = (c0 + c1) + (c2 + c3);
        }
        __syncthreads();
        nloc = 0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            buf[i] = v[nloc++];
            int64_t gi = (base >> (2 * k)) + i;
            if (gi < (cnt >> (2 * k))) dst[gi] = buf[i];
        }
        __syncthreads();
    }
    if (tail > 0) {
        __shared__ unsigned s_last;
        unsigned long long *done = reinterpret_cast<unsigned long long *>(norm2 + 1);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(done, 1ull) == (unsigned long long)(ncta - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        const int top = lf - levels;
        for (int l = top - 1; l >= top - tail; l--) {
            const double *c = norm2 + pyr_off(l + 1);
            double *dst = norm2 + pyr_off(l);
            for (int64_t i = threadIdx.x; i < ((int64_t)1 << (2 * l)); i += blockDim.x) {
                const double c0 = __ldcg(c + 4 * i), c1 = __ldcg(c + 4 * i + 1), c2 = __ldcg(c + 4 * i + 2),
                             c3 = __ldcg(c + 4 * i + 3);
                dst[i] = (c0 + c1) + (c2 + c3);
            }
            __threadfence_block();
            __syncthreads();
        }
        if (threadIdx.x == 0) *done = 0ull;   // the padding is zero again
    }
}

static spamm_status pyramid_kernels(spamm_ctx ctx, spamm_mat m, spamm_mat m2 = nullptr)
{
    int lf = m->L;
    double *n2b = m2 ? m2->norm2 : nullptr;
    while (lf > 0) {
        int lv = lf >= 5 ? 5 : lf;
        const int rest = lf - lv, tail = rest <= 5 ? rest : 0;   // the last CTA finishes <= 5 levels
        int64_t cnt = int64_t(1) << (2 * lf);
        const int grid = cdiv(cnt, int64_t(1) << (2 * lv)), g2 = m2 ? 2 * grid : grid;
        switch (lv) {
        case 5: CK(launch_k(ctx, k_pyramid<5>, g2, 256, 0, m->norm2, lf, 5, tail, n2b, grid)); break;
        case 4: CK(launch_k(ctx, k_pyramid<4>, g2, 256, 0, m->norm2, lf, 4, tail, n2b, grid)); break;
        case 3: CK(launch_k(ctx, k_pyramid<3>, g2, 64, 0, m->norm2, lf, 3, tail, n2b, grid)); break;
        case 2: CK(launch_k(ctx, k_pyramid<2>, g2, 16, 0, m->norm2, lf, 2, tail, n2b, grid)); break;
        default: CK(launch_k(ctx, k_pyramid<1>, g2, 4, 0, m->norm2, lf, 1, tail, n2b, grid)); break;
        }
        CKL(ctx);
        lf -= lv + tail;
    }
    return SPAMM_OK;
}

spamm_status pyramid_build(spamm_ctx ctx, spamm_mat m) { return pyramid_kernels(ctx, m); }
// two pyramids of the same shape in one launch per pass (bitwise the two separate builds)
spamm_status pyramid_build_pair(spamm_ctx ctx, spamm_mat m, spamm_mat m2)
{
    if (m2->L != m->L) return set_err(ctx, SPAMM_EINVAL, "pyramid pair: shapes differ");
    return pyramid_kernels(ctx, m, m2);
}

// ------------------------------------------------------------- build API
static spamm_status build_common(spamm_ctx ctx, BlockSrc src, int64_t count, int64_t n, int b,
                                 spamm_mat *out)
{
    Parts parts;
    ST(mat_parts(ctx, (int)(n / b), &parts));
    const int r0 = ctx->comm ? parts.rs[ctx->comm->rank] : 0;
    const int r1 = ctx->comm ? parts.rs[ctx->comm->rank + 1] : (int)(n / b);
    // 1. per-candidate squared norms
    double *n2 = dalloc<double>(ctx, count);
    int32_t *slot_of = dalloc<int32_t>(ctx, count);
    int ntiles = cdiv(count, 512);
    int32_t *flags = dalloc<int32_t>(ctx, ntiles + 1);
    V1 *agg = dalloc<V1>(ctx, ntiles), *pre = dalloc<V1>(ctx, ntiles);
    spamm_status st = SPAMM_OK;
    int64_t nblk = 0;
    spamm_mat m = nullptr;
    do {
        if (!n2 || !slot_of || !flags || !agg || !pre) {
            st = set_err(ctx, SPAMM_ENOMEM, "build workspace");
            break;
        }
        if (count > 0) {
            k_block_norm2<<<cdiv(count * 32, 256), 256, 0, ctx->stream>>>(src, count, n2);
            ctx->launches++;
            if (cudaMemsetAsync(flags, 0, sizeof(int32_t) * (ntiles + 1), ctx->stream) != cudaSuccess) {
                st = check_cuda(ctx, cudaGetLastError(), "memset");
                break;
            }
            ScanTiles<V1> tiles{flags, agg, pre, flags + ntiles};
            int grid = ntiles < 2 * ctx->sm_count ? ntiles : 2 * ctx->sm_count;
            k_build_scan<512><<<grid, 512, 0, ctx->stream>>>(src, n2, count, r0, r1, tiles, slot_of);
            ctx->launches++;
            // total present = last tile inclusive prefix
            V1 last;
            st = fetch1(ctx, pre + (ntiles - 1), &last, sizeof(V1));
            if (st) break;
            nblk = last.x;
        }
        st = mat_new(ctx, n, b, nblk, &m);
        if (st) break;
        m->nblk = nblk;
        st = mat_reset_pattern(ctx, m);
        if (st) break;
        if (count > 0) {
            k_build_scatter<<<cdiv(count * 32, 256), 256, 0, ctx->stream>>>(
                src, count, slot_of, n2, m->L, m->pool, m->coord, m->slot, m->norm2 + pyr_off(m->L));
            ctx->launches++;
        }
        st = norms_finish(ctx, m);
    } while (0);
    dev_free(ctx, n2, sizeof(double) * count);
    dev_free(ctx, slot_of, sizeof(int32_t) * count);
    dev_free(ctx, flags, sizeof(int32_t) * (ntiles + 1));
    dev_free(ctx, agg, sizeof(V1) * ntiles);
    dev_free(ctx, pre, sizeof(V1) * ntiles);
    if (st) {
        spamm_mat_free(m);
        return st;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        spamm_mat_free(m);
        return check_cuda(ctx, e, "build");
    }
    *out = m;
    return SPAMM_OK;
}

// Stage a possibly-host buffer on the device; *tmp receives a buffer to free.
template <typename T>
static spamm_status stage_in(spamm_ctx ctx, const T *p, int64_t count, const T **dptr, T **tmp)
{
    *tmp = nullptr;
    if (count == 0 || is_device_ptr(p)) {
        *dptr = p;
        return SPAMM_OK;
    }
    T *d = dalloc<T>(ctx, count);
    if (!d) return set_err(ctx, SPAMM_ENOMEM, "staging buffer");
    CK(cudaMemcpyAsync(d, p, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->stream));
    *dptr = d;
    *tmp = d;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_build_tree(spamm_ctx ctx, const double *dense, int64_t n, int64_t ld,
                                         int32_t b, spamm_mat *out)
{
    if (!ctx || !dense || !out) return set_err(ctx, SPAMM_EINVAL, "NULL argument");
    if (ld < n) return set_err(ctx, SPAMM_EINVAL, "ld < n");
    if (b != 16 && b != 32 && b != 64) return set_err(ctx, SPAMM_EINVAL, "b=%d not in {16,32,64}", b);
    if (n < b || n % b) return set_err(ctx, SPAMM_EINVAL, "n not a multiple of b");
    const double *d;
    double *tmp;
    int64_t elems = (n - 1) * ld + n;
    ST(stage_in(ctx, dense, elems, &d, &tmp));
    BlockSrc src{nullptr, nullptr, nullptr, d, ld, b, (int)(n / b)};
    int64_t nb = n / b;
    spamm_status st = build_common(ctx, src, nb * nb, n, b, out);
    dev_free(ctx, tmp, sizeof(double) * elems);
    return st;
}

extern "C" spamm_status spamm_build_tree_blocks(spamm_ctx ctx, int64_t n, int32_t b, int64_t nblocks,
                                                const int32_t *bi, const int32_t *bj,
                                                const double *blocks, spamm_mat *out)
{
    if (!ctx || !out || nblocks < 0 || (nblocks > 0 && (!bi || !bj || !blocks)))
        return set_err(ctx, SPAMM_EINVAL, "NULL argument");
    if (b != 16 && b != 32 && b != 64) return set_err(ctx, SPAMM_EINVAL, "b=%d not in {16,32,64}", b);
    const int32_t *dbi, *dbj;
    const double *dbl;
    int32_t *t1, *t2;
    double *t3;
    ST(stage_in(ctx, bi, nblocks, &dbi, &t1));
    ST(stage_in(ctx, bj, nblocks, &dbj, &t2));
    ST(stage_in(ctx, blocks, nblocks * b * b, &dbl, &t3));
    BlockSrc src{dbi, dbj, dbl, nullptr, b, b, (int)(n / b)};
    spamm_status st = build_common(ctx, src, nblocks, n, b, out);
    dev_free(ctx, t1, sizeof(int32_t) * nblocks);
    dev_free(ctx, t2, sizeof(int32_t) * nblocks);
    dev_free(ctx, t3, sizeof(double) * nblocks * b * b);
    return st;
}

// --------------------------------------------------------------- maps
// op 0: y = x / c ; op 1: y = (x / c + mu delta) / (1 + mu) ; op 2: y = x * c ;
// op 4: y = 1.5 delta - 0.5 x (= 1/2 (3I - X)) ; op 5: y = delta (identity) ;
// op 7: y = x (copy) ; op 8: y = x / c + mu delta (shifted normalised s, regularised
// slices).  Same pattern as src, plus the diagonal for ops 1, 4, 5, 7, 8
// (op 7 adds absent diagonal blocks as zeros, for the scaled map that follows).
// Vectorised map over one stored block per CTA (double2 in the pool layout) with
// the block's squared norm fused in (thread partials in element order, then a
// fixed warp-shuffle + warp-order tree: deterministic).  Same ops as k_map.
__global__ void __launch_bounds__(256) k_map2(const double *src, const int32_t *coord, int b, int op, double c,
                                              double mu, double *dst, double *leaf_n2)
{
    __shared__ double red[8];
    const int64_t blk = blockIdx.x;
    const uint32_t code = coord[blk];
    const bool diag = morton_i(code) == morton_j(code);
    const int64_t base = blk * (int64_t)b * b;
    const double2 *s2 = src ? reinterpret_cast<const double2 *>(src + base) : nullptr;
    double2 *d2 = reinterpret_cast<double2 *>(dst + base);
    const int half = b / 2, n2 = b * b / 2;
    double ss = 0.0;
    for (int p = threadIdx.x; p < n2; p += 256) {
        const int r = p / half, ch = p % half;
        const int q0 = (ch ^ swz(r)) << 1;            // logical column of the pair's first element
        const double2 x = s2 ? s2[p] : make_double2(0.0, 0.0);
        const double dl0 = (diag && r == q0) ? 1.0 : 0.0, dl1 = (diag && r == q0 + 1) ? 1.0 : 0.0;
        double y0, y1;
        switch (op) {
        case 0: y0 = x.x / c; y1 = x.y / c; break;
        case 1: y0 = (x.x / c + mu * dl0) / (1.0 + mu); y1 = (x.y / c + mu * dl1) / (1.0 + mu); break;
        case 2: y0 = x.x * c; y1 = x.y * c; break;
        case 4: y0 = 1.5 * dl0 - 0.5 * x.x; y1 = 1.5 * dl1 - 0.5 * x.y; break;
        case 7: y0 = x.x; y1 = x.y; break;
        case 8: y0 = x.x / c + mu * dl0; y1 = x.y / c + mu * dl1; break;
        default: y0 = dl0; y1 = dl1; break;
        }
        d2[p] = make_double2(y0, y1);
        ss = fma(y0, y0, ss);
        ss = fma(y1, y1, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; w++) t += red[w];
        leaf_n2[code] = t;
    }
}

spamm_status mat_map(spamm_ctx ctx, spamm_mat src, int op, double c, double mu, spamm_mat *out)
{
    bool fill = (op == 1 || op == 4 || op == 5 || op == 7 || op == 8);
    int64_t cap = src->nblk + (fill ? src->nb : 0);
    spamm_mat m;
    ST(mat_new(ctx, src->n, src->b, cap, &m));
    spamm_status st = SPAMM_OK;
    do {
        if (src->nblk > 0) {
            CK(cudaMemcpyAsync(m->slot, src->slot, sizeof(int32_t) * (size_t)src->nb * src->nb,
                               cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaMemcpyAsync(m->coord, src->coord, sizeof(int32_t) * src->nblk,
                               cudaMemcpyDeviceToDevice, ctx->stream));
            CK(cudaMemsetAsync(m->norm2, 0, sizeof(double) * pyr_size(m->L), ctx->stream));
            k_map2<<<(int)src->nblk, 256, 0, ctx->stream>>>(src->pool, src->coord, src->b, op, c, mu, m->pool,
                                                           m->norm2 + pyr_off(m->L));
            CKL(ctx);
        } else {
            CK(cudaMemsetAsync(m->slot, 0xFF, sizeof(int32_t) * (size_t)src->nb * src->nb, ctx->stream));
            CK(cudaMemsetAsync(m->norm2, 0, sizeof(double) * pyr_size(m->L), ctx->stream));
        }
        m->nblk = src->nblk;
        if (fill) {
            // absent diagonal blocks: x = 0 => op 1 gives mu/(1+mu) I, op 4 1.5 I, op 5 I, op 7 0
            double dv = (op == 5) ? 1.0 : (op == 4) ? 1.5 : (op == 7) ? 0.0 : (op == 8) ? mu
                      : (0.0 / c + mu * 1.0) / (1.0 + mu);
            int64_t h = 0;
            st = diag_append(ctx, m, m->nblk, dv, &h);
            if (st) break;
            m->nblk += h;
        }
        st = norms_finish(ctx, m);
    } while (0);
    if (st) {
        spamm_mat_free(m);
        return st;
    }
    *out = m;
    return SPAMM_OK;
}

// ------------------------------------------------------------- readers
__global__ void k_to_dense(const double *pool, const int32_t *coord, int64_t nblk, int b,
                           double *dense, int64_t ld)
{
    int64_t blk = blockIdx.x;
    uint32_t code = coord[blk];
    int I = morton_i(code), J = morton_j(code);
    const double *s = pool + blk * (int64_t)b * b;
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
        int r = e / b, q = pool_col(e, b);
        dense[(int64_t)(I * b + r) * ld + (J * b + q)] = s[e];
    }
}

extern "C" spamm_status spamm_to_dense(spamm_ctx ctx, spamm_mat m, double *dense, int64_t ld)
{
    if (!ctx || !m || !dense || ld < m->n) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    int64_t elems = (m->n - 1) * ld + m->n;
    double *d = dense, *tmp = nullptr;
    bool host = !is_device_ptr(dense);
    if (host) {
        tmp = d = dalloc<double>(ctx, elems);
        if (!d) return set_err(ctx, SPAMM_ENOMEM, "to_dense staging");
    }
    // zero the n x n window (row by row when ld > n)
    if (ld == m->n) CK(cudaMemsetAsync(d, 0, sizeof(double) * elems, ctx->stream));
    else CK(cudaMemset2DAsync(d, ld * sizeof(double), 0, m->n * sizeof(double), m->n, ctx->stream));
    if (m->nblk > 0) {
        k_to_dense<<<(int)m->nblk, 256, 0, ctx->stream>>>(m->pool, m->coord, m->nblk, m->b, d, ld);
        CKL(ctx);
    }
    if (host) {
        CK(cudaMemcpyAsync(dense, d, sizeof(double) * elems, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        dev_free(ctx, tmp, sizeof(double) * elems);
    }
    return SPAMM_OK;
}

__global__ void k_level_rowmajor(const double *lev, int side, double *out)
{
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)side * side) return;
    int I = (int)(e / side), J = (int)(e % side);
    out[e] = lev[morton(I, J)];
}

extern "C" spamm_status spamm_level_norms2(spamm_ctx ctx, spamm_mat m, int32_t level, double *out)
{
    if (!ctx || !m || !out || level < 0 || level > m->L) return set_err(ctx, SPAMM_EINVAL, "bad level");
    int side = 1 << level;
    int64_t cnt = (int64_t)side * side;
    bool host = !is_device_ptr(out);
    double *d = host ? dalloc<double>(ctx, cnt) : out;
    k_level_rowmajor<<<cdiv(cnt, 256), 256, 0, ctx->stream>>>(m->norm2 + pyr_off(level), side, d);
    CKL(ctx);
    if (host) {
        CK(cudaMemcpyAsync(out, d, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        dev_free(ctx, d, sizeof(double) * cnt);
    }
    return SPAMM_OK;
}

__global__ void k_get_blocks(const double *pool, const int32_t *slot, int b, int64_t nreq,
                             const int32_t *bi, const int32_t *bj, double *out, int32_t *present)
{
    int64_t t = blockIdx.x;
    if (t >= nreq) return;
    int s = slot[morton(bi[t], bj[t])];
    double *d = out + t * (int64_t)b * b;
    for (int e = threadIdx.x; e < b * b; e += blockDim.x)
        d[e] = s >= 0 ? pool[(int64_t)s * b * b + pool_at(e / b, e % b, b)] : 0.0;
    if (threadIdx.x == 0 && present) present[t] = s >= 0;
}

extern "C" spamm_status spamm_get_blocks(spamm_ctx ctx, spamm_mat m, int64_t nreq, const int32_t *bi,
                                         const int32_t *bj, double *out, int32_t *present)
{
    if (!ctx || !m || nreq < 0 || (nreq > 0 && (!bi || !bj || !out)))
        return set_err(ctx, SPAMM_EINVAL, "bad argument");
    if (nreq == 0) return SPAMM_OK;
    const int32_t *dbi, *dbj;
    int32_t *t1, *t2;
    ST(stage_in(ctx, bi, nreq, &dbi, &t1));
    ST(stage_in(ctx, bj, nreq, &dbj, &t2));
    int64_t b2 = (int64_t)m->b * m->b;
    bool hout = !is_device_ptr(out);
    bool hpres = present && !is_device_ptr(present);
    double *dout = hout ? dalloc<double>(ctx, nreq * b2) : out;
    int32_t *dpres = hpres ? dalloc<int32_t>(ctx, nreq) : present;
    k_get_blocks<<<(int)nreq, 256, 0, ctx->stream>>>(m->pool, m->slot, m->b, nreq, dbi, dbj, dout, dpres);
    CKL(ctx);
    if (hout) CK(cudaMemcpyAsync(out, dout, sizeof(double) * nreq * b2, cudaMemcpyDeviceToHost, ctx->stream));
    if (hpres) CK(cudaMemcpyAsync(present, dpres, sizeof(int32_t) * nreq, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (hout) dev_free(ctx, dout, sizeof(double) * nreq * b2);
    if (hpres) dev_free(ctx, dpres, sizeof(int32_t) * nreq);
    dev_free(ctx, t1, sizeof(int32_t) * nreq);
    dev_free(ctx, t2, sizeof(int32_t) * nreq);
    return SPAMM_OK;
}

extern "C" spamm_status spamm_mat_info(spamm_mat m, int64_t *n, int32_t *b, int64_t *nblocks)
{
    if (!m) return SPAMM_EINVAL;
    if (n) *n = m->n;
    if (b) *b = m->b;
    if (nblocks) *nblocks = m->nblk;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_norm(spamm_ctx ctx, spamm_mat m, double *fro)
{
    if (!ctx || !m || !fro) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    double r;
    ST(fetch1(ctx, m->norm2, &r, sizeof(double)));
    *fro = sqrt(r);
    return SPAMM_OK;
}

extern "C" spamm_status spamm_scale(spamm_ctx ctx, spamm_mat m, double alpha, int32_t divide,
                                    spamm_mat *out)
{
    if (!ctx || !m || !out) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    return mat_map(ctx, m, divide ? 0 : 2, alpha, 0.0, out);
}

extern "C" spamm_status spamm_ns_y0(spamm_ctx ctx, spamm_mat s, double c, double mu, spamm_mat *Y0)
{
    if (!ctx || !s || !Y0 || !(c > 0.0) || !(mu >= 0.0)) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    return mat_map(ctx, s, mu != 0.0 ? 1 : 0, c, mu, Y0);
}

extern "C" spamm_status spamm_identity(spamm_ctx ctx, int64_t n, int32_t b, spamm_mat *I)
{
    if (!ctx || !I) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    spamm_mat z;
    ST(mat_new(ctx, n, b, 0, &z));
    z->nblk = 0;
    spamm_status st = mat_map(ctx, z, 5, 1.0, 0.0, I);
    spamm_mat_free(z);
    return st;
}
