// power.cu — c ~ ||s||_2 for the spectral rescale s <- s / s_{N-1} (P:380-381,
// "easily obtained largest eigenvalue"; reading L12): K power steps from
// v0 = 1/sqrt(n) * ones, then the Rayleigh quotient c = v^T s v.
// Block-CSR SpMV (one CTA per block row, blocks in ascending column order,
// warp-per-row dot products with fixed-order shuffle reductions: deterministic).
#include <cstdlib>

#include "common.cuh"
#include "scan.cuh"
#include "tma.cuh"

// per block row: count of present blocks
__global__ void k_row_count(const int32_t *slot, int nb, int32_t *cnt)
{
    __shared__ int sh[256];
    int i = blockIdx.x, c = 0;
    for (int j = threadIdx.x; j < nb; j += 256) c += slot[morton(i, j)] >= 0;
    sh[threadIdx.x] = c;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) cnt[i] = sh[0];
}

// single CTA exclusive scan of nb row counts -> rowptr[nb+1]
__global__ void k_row_scan(const int32_t *cnt, int nb, int32_t *rowptr)
{
    __shared__ V1 sw[32];
    int run = 0;
    for (int i0 = 0; i0 < nb; i0 += 1024) {
        int i = i0 + threadIdx.x;
        V1 v{i < nb ? cnt[i] : 0};
        V1 tot;
        V1 ex = block_excl_scan<V1, 1024>(v, &tot, sw);
        if (i < nb) rowptr[i] = run + ex.x;
        run += tot.x;
        __syncthreads();
    }
    if (threadIdx.x == 0) rowptr[nb] = run;
}

// per block row: slots and column indices of present blocks, ascending j
__global__ void k_row_fill(const int32_t *slot, int nb, const int32_t *rowptr, int32_t *cols,
                           int32_t *slots)
{
    __shared__ V1 sw[8];
    int i = blockIdx.x, run = rowptr[i];
    for (int j0 = 0; j0 < nb; j0 += 256) {
        int j = j0 + threadIdx.x;
        int s = j < nb ? slot[morton(i, j)] : -1;
        V1 v{s >= 0 ? 1 : 0};
        V1 tot;
        V1 ex = block_excl_scan<V1, 256>(v, &tot, sw);
        if (s >= 0) {
            cols[run + ex.x] = j;
            slots[run + ex.x] = s;
        }
        run += tot.x;
        __syncthreads();
    }
}

// w[I*b + r] = sum over present blocks (I,J), ascending J, of S_IJ[r,:] . v[J*b:].
// Thread t owns E consecutive (swizzled) elements of one row; TPR = b/E threads
// per row, RG = 256/TPR rows per CTA, b/RG CTAs per block row.  Each thread
// accumulates its partial dot products over the row's blocks in order (U blocks
// in flight), then the TPR threads of a row reduce with a fixed xor tree.
// Persistent: CTAs take (block row, row group) units from a ticket, so the grid is
// exactly the resident capacity (no partial last wave) and uneven rows balance.
template <int B>
__global__ void __launch_bounds__(256) k_spmv(const double *pool, const int32_t *rowptr,
                                              const int32_t *cols, const int32_t *slots,
                                              const double *v, double *w, int32_t *ticket, int nunits)
{
    constexpr int E = B >= 32 ? 4 : 1, TPR = B / E, RG = 256 / TPR, CPR = B / RG;
    __shared__ int s_unit;
    for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(ticket, 1);
    __syncthreads();
    const int unit = s_unit;
    __syncthreads();
    if (unit >= nunits) return;
    const int I = unit / CPR, rg = unit % CPR;
    const int p0 = rowptr[I], p1 = rowptr[I + 1];
    const int r = rg * RG + threadIdx.x / TPR;
    const int e0 = r * B + (threadIdx.x % TPR) * E;   // physical offset inside a block
    int lc[E];
#pragma unroll
    for (int i = 0; i < E; i++) lc[i] = pool_col(e0 + i, B);
    double acc = 0.0;
    constexpr int U = 4;      // blocks in flight per thread
    constexpr int SPC = 512;  // block-row entries staged in shared memory per pass
    __shared__ int s_slot[SPC], s_col[SPC];
    for (int pc = p0; pc < p1; pc += SPC) {
        const int pe = p1 < pc + SPC ? p1 : pc + SPC;
        __syncthreads();
        for (int i = threadIdx.x; i < pe - pc; i += 256) {
            s_slot[i] = slots[pc + i];
            s_col[i] = cols[pc + i];
        }
        __syncthreads();
        // one global round trip per U blocks: the slot / column indices come from smem
        for (int p = pc; p < pe; p += U) {
            double x[U][E], vx[U][E];
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (p + u < pe) {
                    const double *blk = pool + (int64_t)s_slot[p + u - pc] * B * B + e0;
                    const double *vv = v + (int64_t)s_col[p + u - pc] * B;
                    if constexpr (E >= 2) {
#pragma unroll
                        for (int i = 0; i < E; i += 2) {
                            double2 t = __ldg(reinterpret_cast<const double2 *>(blk + i));
                            x[u][i] = t.x;
                            x[u][i + 1] = t.y;
                        }
                    } else {
                        x[u][0] = __ldg(blk);
                    }
#pragma unroll
                    for (int i = 0; i < E; i++) vx[u][i] = __ldg(vv + lc[i]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (p + u < pe) {
                    double sdot = 0.0;
#pragma unroll
                    for (int i = 0; i < E; i++) sdot = fma(x[u][i], vx[u][i], sdot);
                    acc += sdot;
                }
            }
        }
    }
#pragma unroll
    for (int o = 1; o < TPR; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x % TPR) == 0) w[(int64_t)I * B + r] = acc;
    }
}

// ------------------------------------------------- TMA-staged SpMV (b = 64)
// One persistent CTA per SM streams whole 32 KiB blocks into a 6-stage shared
// memory ring with TMA bulk copies (thread 0 issues, mbarrier transaction counts
// signal arrival), so ~192 KiB per SM are in flight without holding them in
// registers.  Work units are quarters of block rows (a quarter of the row's blocks,
// ascending), taken from a ticket; a thread owns one 16-byte chunk of 8 rows of
// each block (consecutive lanes read consecutive chunks: conflict-free) and keeps
// 8 row accumulators across the unit's blocks.  Each unit writes its 64 partial row
// sums; k_spmv_fix adds the 4 quarters in a fixed order (deterministic).
constexpr int SPT_Q = 4;                       // work unit = a quarter of a block row
// stages of the ring per leaf size: 6 x 32 KiB (b=64), 16 x 8 KiB (b=32), 32 x 2 KiB (b=16)
template <int B> struct SptCfg {
    static constexpr int STAGES = B == 64 ? 6 : B == 32 ? 16 : 32;
    static constexpr int LPR = B / 2;           // lanes (double2 chunks) per block row
    static constexpr int N2 = B * B / 2;        // double2 per block
    static constexpr int M = (N2 + 255) / 256;  // double2 per thread per block (256 threads)
    static constexpr int RPW = 32 / LPR;        // block rows per warp per m
};

struct SpmvTmaArgs {
    const double *pool;
    const int32_t *rowptr, *cols, *slots;
    const double *v;
    double *part;       // [nb * SPT_Q * b]
    int32_t *ticket;
    int nunits;         // nb * SPT_Q
};

template <int B>
__global__ void __launch_bounds__(256, 1) k_spmv_tma(SpmvTmaArgs g)
{
    using Cf = SptCfg<B>;
    constexpr int TILE = B * B, STAGES = Cf::STAGES, LPR = Cf::LPR, M = Cf::M, RPW = Cf::RPW, N2 = Cf::N2;
    extern __shared__ __align__(1024) double sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + STAGES * TILE);
    int4 *meta = reinterpret_cast<int4 *>(full + STAGES);   // {unit, column block, last, -}
    __shared__ int s_total;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // issuer state (thread 0); the unit's slot / column indices are fetched in one
    // batch of independent loads (UCH at a time), not one dependent load per issue
    constexpr int UCH = 32;
    int issued = 0, unit = -1, p = 0, pend = 0, ubase = 0;
    int us[UCH], uc[UCH];
    bool done = false;
    if (tid == 0) {
        for (int st = 0; st < STAGES; st++) mbar_init(&full[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        s_total = -1;
    }
    __syncthreads();
    // thread tid owns double2 chunk q = tid + 256 m of each block: block row
    // q / LPR, chunk q % LPR (consecutive lanes, consecutive 16 B: conflict-free)
    double acc[M];
    int lc[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int q = tid + 256 * m, r = q / LPR;
        acc[m] = 0.0;
        lc[m] = ((q % LPR) ^ swz(r)) << 1;   // logical column pair (pool swizzle)
    }
    for (int j = 0;; j++) {
        if (tid == 0) {
            // keep the ring full: blocks j .. j + STAGES - 1 in flight
            while (!done && issued < j + STAGES) {
                if (p == pend) {
                    unit = atomicAdd(g.ticket, 1);
                    if (unit >= g.nunits) {
                        done = true;
                        s_total = issued;
                        break;
                    }
                    const int I = unit / SPT_Q, q = unit % SPT_Q;
                    const int p0 = g.rowptr[I], len = g.rowptr[I + 1] - p0;
                    p = p0 + (q * len) / SPT_Q;
                    pend = p0 + ((q + 1) * len) / SPT_Q;
                    ubase = p - UCH;   // forces a fetch below
                    continue;
                }
                if (p - ubase >= UCH) {
                    ubase = p;
#pragma unroll
                    for (int i = 0; i < UCH; i++) {
                        us[i] = p + i < pend ? __ldg(g.slots + p + i) : 0;
                        uc[i] = p + i < pend ? __ldg(g.cols + p + i) : 0;
                    }
                }
                const int st = issued % STAGES;
                meta[st] = make_int4(unit, uc[p - ubase], p + 1 == pend, 0);
                mbar_expect_tx(&full[st], TILE * 8);
                bulk_g2s(sm + st * TILE, g.pool + (int64_t)us[p - ubase] * TILE, TILE * 8, &full[st]);
                issued++;
                p++;
            }
        }
        __syncthreads();
        if (s_total >= 0 && j >= s_total) break;
        const int st = j % STAGES;
        mbar_wait(&full[st], (j / STAGES) & 1);
        const int4 mt = meta[st];
        const double2 *x2 = reinterpret_cast<const double2 *>(sm + st * TILE);
        const double *vv = g.v + (int64_t)mt.y * B;
#pragma unroll
        for (int m = 0; m < M; m++) {
            if (tid + 256 * m >= N2) break;      // b = 16: warps 4..7 idle (warp-uniform)
            const double2 x = x2[tid + 256 * m];
            const double2 w = *reinterpret_cast<const double2 *>(vv + lc[m]);
            acc[m] = fma(x.x, w.x, acc[m]);
            acc[m] = fma(x.y, w.y, acc[m]);
        }
        if (mt.z) {
            // last block of the unit: each block row's LPR lanes reduce with a fixed xor tree
#pragma unroll
            for (int m = 0; m < M; m++) {
                if (tid + 256 * m >= N2) break;
                double t = acc[m];
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (lane % LPR == 0)
                    g.part[(int64_t)mt.x * B + (warp * RPW + lane / LPR) + (256 / LPR) * m] = t;
                acc[m] = 0.0;
            }
        }
        __syncthreads();   // stage st may be refilled from the next iteration on
    }
}

// w[I*b + r] = (P0 + P1) + (P2 + P3), P_q = quarter q's partial (0 if the quarter is empty)
__global__ void k_spmv_fix(const int32_t *rowptr, const double *part, int nb, int b, double *w)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)nb * b) return;
    const int I = (int)(e / b), r = (int)(e % b);
    const int p0 = rowptr[I], len = rowptr[I + 1] - p0;
    double P[SPT_Q];
#pragma unroll
    for (int q = 0; q < SPT_Q; q++) {
        const bool any = ((q + 1) * len) / SPT_Q > (q * len) / SPT_Q;
        P[q] = any ? part[((int64_t)I * SPT_Q + q) * b + r] : 0.0;
    }
    w[e] = (P[0] + P[1]) + (P[2] + P[3]);
}

// single CTA: nrm = sqrt(sum w^2) (fixed order); v = w / nrm
__global__ void k_normalize(const double *w, int64_t n, double *v)
{
    __shared__ double sh[1024];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 1024) s = fma(w[i], w[i], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int k = 512; k > 0; k >>= 1) {
        if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    double nrm = sqrt(sh[0]);
    for (int64_t i = threadIdx.x; i < n; i += 1024) v[i] = w[i] / nrm;
}

// Large n: the normalisation in two launches over NRM_CTAS contiguous chunks
// (partials in chunk order, then every CTA sums the partials in the same order,
// so all agree bitwise on the norm) instead of one CTA streaming all of w.
constexpr int NRM_CTAS = 128;
__global__ void __launch_bounds__(256) k_sumsq_part(const double *w, int64_t n, double *part)
{
    __shared__ double sh[256];
    const int64_t chunk = (n + NRM_CTAS - 1) / NRM_CTAS, i0 = blockIdx.x * chunk;
    const int64_t i1 = i0 + chunk < n ? i0 + chunk : n;
    double s = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += 256) s = fma(w[i], w[i], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) k_scale_by_norm(const double *w, int64_t n, const double *part, double *v)
{
    __shared__ double nrm;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int c = 0; c < NRM_CTAS; c++) t += part[c];
        nrm = sqrt(t);
    }
    __syncthreads();
    const int64_t chunk = (n + NRM_CTAS - 1) / NRM_CTAS, i0 = blockIdx.x * chunk;
    const int64_t i1 = i0 + chunk < n ? i0 + chunk : n;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += 256) v[i] = w[i] / nrm;
}

__global__ void k_fill(double *v, int64_t n, double val)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = val;
}

__global__ void k_dot(const double *a, const double *b, int64_t n, double *out)
{
    __shared__ double sh[1024];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 1024) s = fma(a[i], b[i], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int k = 512; k > 0; k >>= 1) {
        if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

template <int B>
static spamm_status spmv_tma(spamm_ctx ctx, spamm_mat s, const int32_t *rowptr, const int32_t *cols,
                             const int32_t *slots, const double *v, double *w, int32_t *ticket, double *part)
{
    constexpr int STAGES = SptCfg<B>::STAGES;
    const size_t smem = sizeof(double) * STAGES * B * B + STAGES * (sizeof(uint64_t) + sizeof(int4));
    static std::atomic<uint64_t> configured{0};
    CK(once_per_device(configured, ctx->device, [&]() {
        return cudaFuncSetAttribute(k_spmv_tma<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }));
    SpmvTmaArgs g{s->pool, rowptr, cols, slots, v, part, ticket, s->nb * SPT_Q};
    k_spmv_tma<B><<<ctx->sm_count, 256, smem, ctx->stream>>>(g);
    CKL(ctx);
    k_spmv_fix<<<cdiv((int64_t)s->nb * B, 256), 256, 0, ctx->stream>>>(rowptr, part, s->nb, B, w);
    CKL(ctx);
    return SPAMM_OK;
}

template <int B>
static void spmv(spamm_ctx ctx, spamm_mat s, const int32_t *rowptr, const int32_t *cols,
                 const int32_t *slots, const double *v, double *w, int32_t *ticket)
{
    constexpr int E = B >= 32 ? 4 : 1, TPR = B / E, RG = 256 / TPR, CPR = B / RG;
    static std::atomic<int> occ_cache{0};
    int occ = occ_cache.load();
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv<B>, 256, 0);
        if (occ < 1) occ = 1;
        occ_cache.store(occ);
    }
    const int nunits = s->nb * CPR;
    int grid = ctx->sm_count * occ;
    if (grid > nunits) grid = nunits;
    k_spmv<B><<<grid, 256, 0, ctx->stream>>>(s->pool, rowptr, cols, slots, v, w, ticket, nunits);
    ctx->launches++;
}

// SPAMM_SPMV_TMA=0 selects the register-streaming SpMV (k_spmv) instead
static bool spmv_tma_mode()
{
    // function-local static: initialised once, thread-safely (C++11)
    static const bool m = [] {
        const char *e = getenv("SPAMM_SPMV_TMA");
        return !(e && *e == '0');
    }();
    return m;
}

spamm_status power_scale(spamm_ctx ctx, spamm_mat s, int K, double *c_host)
{
    const int nb = s->nb;
    const int64_t n = s->n;
    int64_t nblk = s->nblk > 0 ? s->nblk : 1;
    int32_t *cnt = dalloc<int32_t>(ctx, nb), *rowptr = dalloc<int32_t>(ctx, nb + 1);
    int32_t *cols = dalloc<int32_t>(ctx, nblk), *slots = dalloc<int32_t>(ctx, nblk);
    double *v = dalloc<double>(ctx, n), *w = dalloc<double>(ctx, n);
    double *c = dalloc<double>(ctx, 1 + NRM_CTAS);   // [0] = c, [1..] normalisation partials
    int32_t *tickets = dalloc<int32_t>(ctx, K + 1);   // one per SpMV launch
    // TMA staging pays for 32 KiB blocks; for b = 16 / 32 the per-block barrier of the
    // ring dominates (C2 setup 4.3 -> 8.4 ms measured), so those keep the register kernel
    const bool tma = spmv_tma_mode() && s->b == 64;
    double *part = tma ? dalloc<double>(ctx, (int64_t)nb * SPT_Q * s->b) : nullptr;
    if (!cnt || !rowptr || !cols || !slots || !v || !w || !c || !tickets || (tma && !part))
        return set_err(ctx, SPAMM_ENOMEM, "power");
    CK(cudaMemsetAsync(tickets, 0, sizeof(int32_t) * (K + 1), ctx->stream));
    int nmv = 0;
    cudaStream_t st = ctx->stream;
    k_row_count<<<nb, 256, 0, st>>>(s->slot, nb, cnt);
    k_row_scan<<<1, 1024, 0, st>>>(cnt, nb, rowptr);
    k_row_fill<<<nb, 256, 0, st>>>(s->slot, nb, rowptr, cols, slots);
    k_fill<<<cdiv(n, 256), 256, 0, st>>>(v, n, 1.0 / sqrt((double)n));
    ctx->launches += 4;
    // row partition: local block rows of w = s v, then all ranks gather the full w
    // (each row is computed by one rank with the single-device kernel: bitwise G-invariant)
    auto mv = [&](const double *x, double *y) -> spamm_status {
        int32_t *tk = tickets + nmv++;
        if (tma) {
            switch (s->b) {
            case 16: ST(spmv_tma<16>(ctx, s, rowptr, cols, slots, x, y, tk, part)); break;
            case 32: ST(spmv_tma<32>(ctx, s, rowptr, cols, slots, x, y, tk, part)); break;
            default: ST(spmv_tma<64>(ctx, s, rowptr, cols, slots, x, y, tk, part)); break;
            }
            return s->dist ? gather_rows(ctx, s->parts, y, s->b) : SPAMM_OK;
        }
        switch (s->b) {
        case 16: spmv<16>(ctx, s, rowptr, cols, slots, x, y, tk); break;
        case 32: spmv<32>(ctx, s, rowptr, cols, slots, x, y, tk); break;
        default: spmv<64>(ctx, s, rowptr, cols, slots, x, y, tk); break;
        }
        return s->dist ? gather_rows(ctx, s->parts, y, s->b) : SPAMM_OK;
    };
    for (int it = 0; it < K; it++) {
        ST(mv(v, w));
        if (n >= (1 << 16)) {
            k_sumsq_part<<<NRM_CTAS, 256, 0, st>>>(w, n, c + 1);
            k_scale_by_norm<<<NRM_CTAS, 256, 0, st>>>(w, n, c + 1, v);
            ctx->launches++;
        } else {
            k_normalize<<<1, 1024, 0, st>>>(w, n, v);
        }
        ctx->launches++;
    }
    ST(mv(v, w));
    k_dot<<<1, 1024, 0, st>>>(v, w, n, c);
    CKL(ctx);
    double h = 0;
    ST(fetch1(ctx, c, &h, sizeof(double)));
    *c_host = h;
    dev_free(ctx, cnt, sizeof(int32_t) * nb);
    dev_free(ctx, rowptr, sizeof(int32_t) * (nb + 1));
    dev_free(ctx, cols, sizeof(int32_t) * nblk);
    dev_free(ctx, slots, sizeof(int32_t) * nblk);
    dev_free(ctx, v, sizeof(double) * n);
    dev_free(ctx, w, sizeof(double) * n);
    dev_free(ctx, c, sizeof(double) * (1 + NRM_CTAS));
    dev_free(ctx, tickets, sizeof(int32_t) * (K + 1));
    dev_free(ctx, part, sizeof(double) * (int64_t)nb * SPT_Q * s->b);
    return SPAMM_OK;
}
