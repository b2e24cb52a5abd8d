// power.cu — c ~ ||s||_2 for the spectral rescale s <- s / s_{N-1} (P:380-381,
// "easily obtained largest eigenvalue"; reading L12): K power steps from
// v0 = 1/sqrt(n) * ones, v <- w / ||w||, w = s v, then the Rayleigh quotient
// c = v^T s v.  Block-CSR SpMV over the pool, every sum in a fixed order
// (deterministic, no atomics):
//   b = 64 : k_spmv_tma<64, SYM> — persistent, warp-specialised TMA ring; with s
//            checked bitwise symmetric (k_sym_check) only the blocks on and above
//            the block diagonal are read (SYM), the rest via column sums;
//   b = 32 : k_spmv_blk<32, SYM> — persistent, one warp per staged block, every block's
//            row (and, SYM, column) part stored on its own and summed per row by
//            k_spmv_bfix in CSR order; the normalisation folded into the next SpMV
//            (C2: 3.12 -> 2.01 ms per power iteration);
//   b = 16 : k_spmv — register streaming (C1, n = 256, is launch-bound).
// Consecutive SpMVs take their work units in opposite orders (zig-zag, L2 reuse).
#include <cstdlib>

#include <cooperative_groups.h>

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
// per row, RG = NT/TPR rows per CTA, b/RG CTAs per block row.  Each thread
// accumulates its partial dot products over the row's blocks in order (U blocks
// in flight), then the TPR threads of a row reduce with a fixed xor tree.  A row's
// arithmetic depends on neither NT nor U.
// Persistent: CTAs take (block row, row group) units from a ticket, so the grid is
// exactly the resident capacity (no partial last wave) and uneven rows balance.
template <int B, int NT>
__global__ void __launch_bounds__(NT) k_spmv(const double *pool, const int32_t *rowptr,
                                             const int32_t *cols, const int32_t *slots,
                                             const double *v, double *w, int32_t *ticket, int nunits,
                                             int rev)
{
    pdl_wait();
    pdl_trigger();
    constexpr int E = B >= 32 ? 4 : 1, TPR = B / E, RG = NT / TPR, CPR = B / RG;
    __shared__ int s_unit;
    for (;;) {
    if (threadIdx.x == 0) s_unit = atomicAdd(ticket, 1);
    __syncthreads();
    const int tk = s_unit;
    __syncthreads();
    if (tk >= nunits) return;
    const int unit = rev ? nunits - 1 - tk : tk;   // zig-zag over the power steps (see power_scale)
    const int I = unit / CPR, rg = unit % CPR;
    const int p0 = rowptr[I], p1 = rowptr[I + 1];
    const int r = rg * RG + threadIdx.x / TPR;
    const int e0 = r * B + (threadIdx.x % TPR) * E;   // physical offset inside a block
    int lc[E];
#pragma unroll
    for (int i = 0; i < E; i++) lc[i] = pool_col(e0 + i, B);
    double acc = 0.0;
    // blocks in flight per thread: ~32-64 KB of loads in flight per CTA, what an SM needs
    // to stream s near the HBM rate (U = 16 with v staged in shared memory measured the
    // same at C2, 3.015 vs 3.017 ms per power iteration)
    constexpr int U = B == 16 ? 16 : 8;
    constexpr int SPC = 512;  // block-row entries staged in shared memory per pass
    __shared__ int s_slot[SPC], s_col[SPC];
    for (int pc = p0; pc < p1; pc += SPC) {
        const int pe = p1 < pc + SPC ? p1 : pc + SPC;
        __syncthreads();
        for (int i = threadIdx.x; i < pe - pc; i += NT) {
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

// ------------------------------------------------- TMA-staged SpMV configuration
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
    int nupper;         // nb * SPT_Q units over the upper parts of the block rows
    int nunits;         // nupper (SYM) or nupper + nb (the lower parts, one unit per row)
    int rev;            // units in descending order (zig-zag over the power steps)
};

// ------------------------------------------------- TMA-staged SpMV kernel
// One persistent CTA per SM streams whole blocks into a shared-memory ring with TMA
// bulk copies.  Warp 8 is the producer: its lane 0 takes work units from a ticket,
// reads the unit's slot / column indices in batches and refills stage st as soon
// as the 8 consumer warps have released it (empty[st]); the consumers never wait
// for the producer's index loads or ticket atomics, only for data (full[st]).
// Consumer thread t owns double2 chunk q = t + 256 m of each block (consecutive
// lanes, consecutive 16 B: conflict-free) and keeps its row accumulators across
// the unit's blocks; at the unit's last block each block row's LPR lanes reduce with
// a fixed xor tree into part[unit*b + r], and k_spmv_sym_fix adds the SPT_Q quarters
// and the column parts in a fixed order (deterministic).  Units: quarters of each
// row's upper part [up[I], rowptr[I+1]) (the blocks on and above the diagonal), and,
// without SYM, one unit per row for its lower part, whose blocks yield column parts
// (below) instead of row sums.
//
// SYM (s symmetric, checked bitwise by k_sym_check): only the upper units run — half
// the HBM reads.  An off-diagonal block (I, J) also contributes S_IJ^T v_I to the rows
// of J: a second pass over the staged tile forms the column sums sum_r S_IJ[r,c] v_I[r]
// (NSUB row subsets per column, reduced in a fixed order after a consumer-only named
// barrier) and stores them at colpart[p'*b ..], p' = the CSR position of the mirror
// (J, I), so k_spmv_sym_fix reads the column parts of row block J contiguously,
// ascending I.  Without SYM the lower block (J, I) itself yields that column part,
// sum_r S_JI[c, r] v_I[r] in the same order: for a symmetric s the two kernels (and
// the row-partitioned path, which has only its own rows) give w bit for bit.
template <int B, bool SYM>
__global__ void __launch_bounds__(288, 1) k_spmv_tma(SpmvTmaArgs g, const int32_t *up, const int32_t *mir,
                                                          double *colpart)
{
    pdl_wait();
    pdl_trigger();
    using Cf = SptCfg<B>;
    constexpr int TILE = B * B, STAGES = Cf::STAGES, LPR = Cf::LPR, M = Cf::M, RPW = Cf::RPW, N2 = Cf::N2;
    constexpr int NSUB = 256 / B, RS = B / NSUB;   // column pass: row subsets, rows per subset
    extern __shared__ __align__(1024) double sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + STAGES * TILE);
    uint64_t *empty = full + STAGES;
    int4 *meta = reinterpret_cast<int4 *>(empty + STAGES);   // {unit (-1: end), column block, last, colpart pos}
    __shared__ double red[2][NSUB][B];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int st = 0; st < STAGES; st++) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {   // ---------------------------------------------- producer
        if (lane != 0) return;
        constexpr int UCH = 32;
        int issued = 0;
        for (;;) {
            const int tk = atomicAdd(g.ticket, 1);
            if (tk >= g.nunits) break;
            const int unit = g.rev ? g.nunits - 1 - tk : tk;
            int pb, pend;
            if (unit < g.nupper) {   // a quarter of the row's upper part [up[I], rowptr[I+1])
                const int I = unit / SPT_Q, q = unit % SPT_Q;
                const int r0 = up[I], len = g.rowptr[I + 1] - r0;
                pb = r0 + (q * len) / SPT_Q;
                pend = r0 + ((q + 1) * len) / SPT_Q;
            } else {                 // (!SYM) the row's lower part [rowptr[I], up[I])
                const int I = unit - g.nupper;
                pb = g.rowptr[I];
                pend = up[I];
            }
            for (int p0 = pb; p0 < pend; p0 += UCH) {
                int us[UCH], uc[UCH], um[UCH];
#pragma unroll
                for (int i = 0; i < UCH; i++) {
                    us[i] = p0 + i < pend ? __ldg(g.slots + p0 + i) : 0;
                    uc[i] = p0 + i < pend ? __ldg(g.cols + p0 + i) : 0;
                    // column-part position: the mirror (SYM) or the lower block itself (!SYM)
                    um[i] = p0 + i < pend ? (SYM ? __ldg(mir + p0 + i) : p0 + i) : 0;
                }
#pragma unroll 1
                for (int i = 0; i < UCH && p0 + i < pend; i++) {
                    const int st = issued % STAGES;
                    if (issued >= STAGES) mbar_wait(&empty[st], ((issued / STAGES) - 1) & 1);
                    meta[st] = make_int4(unit, uc[i], p0 + i + 1 == pend, um[i]);
                    mbar_expect_tx(&full[st], TILE * 8);
                    bulk_g2s(sm + st * TILE, g.pool + (int64_t)us[i] * TILE, TILE * 8, &full[st]);
                    issued++;
                }
            }
        }
        const int st = issued % STAGES;   // end marker
        if (issued >= STAGES) mbar_wait(&empty[st], ((issued / STAGES) - 1) & 1);
        meta[st] = make_int4(-1, 0, 0, 0);
        mbar_arrive(&full[st]);
        return;
    }
    // ----------------------------------------------------------------- consumers
    const int cc = tid % B, sub = tid / B;   // column pass: column, row subset
    double acc[M];
    int lc[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int q = tid + 256 * m, r = q / LPR;
        acc[m] = 0.0;
        lc[m] = ((q % LPR) ^ swz(r)) << 1;   // logical column pair (pool swizzle)
    }
    int vunit = -1, nred = 0;
    double vi[RS];   // v at this thread's column-pass rows
    for (int j = 0;; j++) {
        const int st = j % STAGES;
        mbar_wait(&full[st], (j / STAGES) & 1);
        const int4 mt = meta[st];
        if (mt.x < 0) break;
        const double *tile = sm + st * TILE;
        const double2 *x2 = reinterpret_cast<const double2 *>(tile);
        const double *vv = g.v + (int64_t)mt.y * B;
        const bool lower = !SYM && mt.x >= g.nupper;   // CTA-uniform
        const int I = lower ? mt.x - g.nupper : mt.x / SPT_Q;
        const bool offdiag = SYM && mt.y != I;
        if (!lower) {
#pragma unroll
            for (int m = 0; m < M; m++) {
                if (tid + 256 * m >= N2) break;      // b = 16: warps 4..7 idle (warp-uniform)
                const double2 x = x2[tid + 256 * m];
                const double2 w = *reinterpret_cast<const double2 *>(vv + lc[m]);
                acc[m] = fma(x.x, w.x, acc[m]);
                acc[m] = fma(x.y, w.y, acc[m]);
            }
        }
        if (offdiag) {
            // upper block (I, J): column sums sum_r S_IJ[r, c] v_I[r] for row block J
            if (mt.x != vunit) {
                vunit = mt.x;
#pragma unroll
                for (int i = 0; i < RS; i++) vi[i] = g.v[(int64_t)I * B + sub * RS + i];
            }
            double cs = 0.0;
#pragma unroll
            for (int i = 0; i < RS; i++) cs = fma(tile[pool_at(sub * RS + i, cc, B)], vi[i], cs);
            red[nred & 1][sub][cc] = cs;
        }
        if (lower) {
            // lower block (I, J), J < I: the same sums from the block itself,
            // sum_r S_IJ[c, r] v_J[r] in the column pass's order, so that for a
            // symmetric s this equals the SYM kernel's column part bit for bit
#pragma unroll
            for (int i = 0; i < RS; i++) vi[i] = vv[sub * RS + i];
            double cs = 0.0;
#pragma unroll
            for (int i = 0; i < RS; i++) cs = fma(tile[pool_at(cc, sub * RS + i, B)], vi[i], cs);
            red[nred & 1][sub][cc] = cs;
        }
        if (mt.z && !lower) {
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
        // generic-proxy reads of stage st before its async-proxy (TMA) refill
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (offdiag || lower) {
            asm volatile("bar.sync 1, 256;\n" ::: "memory");   // consumers only: red[nred & 1] complete
            if (tid < B) {
                double t = red[nred & 1][0][tid];
#pragma unroll
                for (int s2 = 1; s2 < NSUB; s2++) t += red[nred & 1][s2][tid];
                colpart[(int64_t)mt.w * B + tid] = t;
            }
            nred++;
        }
    }
}

// Sum of w^2 over the CTA's 256 threads in a fixed order (xor tree in each warp,
// then the 8 warp sums in warp order): the normalisation's partial for this CTA.
__device__ __forceinline__ void cta_sumsq_part(double x, double *nrm_part)
{
    __shared__ double ws[8];
    double t = x * x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double u = ws[0];
        for (int k = 1; k < 8; k++) u += ws[k];
        nrm_part[blockIdx.x] = u;
    }
}

// ------------------------------------------------- per-block SpMV (b = 32 / 16)
// The TMA ring above keeps row accumulators across a unit's blocks, and its column pass needs
// a CTA barrier per block; on 8 / 2 KiB blocks those per-block synchronisations cost more than
// the data (C2: 34 us per pass with s in L2).  Here every block is handled by ONE warp from its
// own shard of the ring, and every block's results are stored on their own, so no warp waits
// for another:
//   row pass     t[r] = sum_c S_IJ[r, c] v_J[c]   (c ascending)  -> bpart[p],    p = (I, J)
//   column pass  u[c] = sum_r S_IJ[r, c] v_I[r]   (r ascending)  -> bpart[p'],   p' = (J, I)
// (the column pass only with SYM, for the blocks above the diagonal; then only those blocks
// are read: s of C2 is 132 MB, its upper half fits in L2).  k_spmv_bfix then forms
// w_J = sum over the CSR positions p of row J, ascending, of bpart[p].  Without SYM (an
// asymmetric s, or the row partition, whose ranks hold only their own rows) every block gets
// the row pass; for a lower block (J, I) that is sum_c S_JI[c', c] v_I[c] = the column pass
// of its mirror term by term, so all paths give w bit for bit.
// Warp w of a CTA takes the CTA's blocks w, w + 8, ... from its shard of BRS stages; a block's
// position in the CTA's stream does not enter its arithmetic (results are deterministic).
#ifndef SPAMM_SPB_VTMA
#define SPAMM_SPB_VTMA 0   // 1: the vector segments staged with the block by bulk copies (C2: 2.38 vs 2.01 ms per power iteration with __ldg)
#endif
template <int B> struct SpbCfg {
    static constexpr int BRS = B == 32 ? 3 : 8;        // stages per consumer warp
    static constexpr int NST = 8 * BRS;
    static constexpr int SD = B * B + 2 * B;            // a stage: the block, then x_J, x_I
    static constexpr size_t smem = sizeof(double) * (NST * SD + 8 * 2 * B) +
                                   NST * (2 * sizeof(uint64_t) + sizeof(int4));
};

// x: the input vector; nrm_part (nullable, single device): x is the previous w and the
// vector is v = x / sqrt(sum of the np partials), the norm formed by every CTA exactly as
// k_norm_apply forms it (so v is bitwise the vector k_norm_apply would have written).
template <int B, bool SYM>
__global__ void __launch_bounds__(288, 1) k_spmv_blk(SpmvTmaArgs g, const int32_t *up, const int32_t *mir,
                                                     double *bpart, const double *nrm_part, int np)
{
    pdl_wait();
    pdl_trigger();
    using Cf = SpbCfg<B>;
    constexpr int TILE = B * B, BRS = Cf::BRS, NST = Cf::NST, SD = Cf::SD;
    extern __shared__ __align__(1024) double sm[];
    double *vbuf = sm + NST * SD;                                     // [8][2][B]: v_J, v_I per warp
    uint64_t *full = reinterpret_cast<uint64_t *>(vbuf + 8 * 2 * B);
    uint64_t *empty = full + NST;
    int4 *meta = reinterpret_cast<int4 *>(empty + NST);               // {p (-1: end), I, J, mirror p'}
    __shared__ double red[256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int st = 0; st < NST; st++) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {   // ---------------------------------------------- producer
        int issued = 0;
        // stage of the CTA's block number i: shard i % 8, slot (i / 8) % BRS
        auto slot = [&](int i, int &st, uint32_t &ph) {
            const int k = i >> 3;
            st = (i & 7) * BRS + k % BRS;
            ph = (uint32_t)((k / BRS) & 1);
        };
        for (;;) {
            int tk = 0;
            if (lane == 0) tk = atomicAdd(g.ticket, 1);
            tk = __shfl_sync(0xffffffffu, tk, 0);
            if (tk >= g.nunits) break;
            const int unit = g.rev ? g.nunits - 1 - tk : tk;
            const int I = unit / SPT_Q, q = unit % SPT_Q;
            const int r0 = SYM ? up[I] : g.rowptr[I], len = g.rowptr[I + 1] - r0;
            const int pb = r0 + (q * len) / SPT_Q, pend = r0 + ((q + 1) * len) / SPT_Q;
            for (int p0 = pb; p0 < pend; p0 += 32) {
                // the indices of up to 32 blocks, one per lane, then lane 0 issues them
                const int p = p0 + lane;
                const int sl = p < pend ? __ldg(g.slots + p) : 0, J = p < pend ? __ldg(g.cols + p) : 0;
                const int pm = p < pend ? (SYM ? __ldg(mir + p) : p) : 0;
                const int cnt = pend - p0 < 32 ? pend - p0 : 32;
                for (int j = 0; j < cnt; j++) {
                    const int slj = __shfl_sync(0xffffffffu, sl, j), Jj = __shfl_sync(0xffffffffu, J, j);
                    const int pmj = __shfl_sync(0xffffffffu, pm, j);
                    if (lane == 0) {
                        int st;
                        uint32_t ph;
                        slot(issued, st, ph);
                        if (issued >= NST) mbar_wait(&empty[st], ph ^ 1);
                        meta[st] = make_int4(p0 + j, I, Jj, pmj);
                        const bool cp = SYM && Jj != I;
                        double *d = sm + st * SD;
                        if (SPAMM_SPB_VTMA) {
                            mbar_expect_tx(&full[st], (TILE + (cp ? 2 : 1) * B) * 8);
                            bulk_g2s(d, g.pool + (int64_t)slj * TILE, TILE * 8, &full[st]);
                            bulk_g2s(d + TILE, g.v + (int64_t)Jj * B, B * 8, &full[st]);
                            if (cp) bulk_g2s(d + TILE + B, g.v + (int64_t)I * B, B * 8, &full[st]);
                        } else {
                            mbar_expect_tx(&full[st], TILE * 8);
                            bulk_g2s(d, g.pool + (int64_t)slj * TILE, TILE * 8, &full[st]);
                        }
                    }
                    issued++;
                }
            }
        }
        if (lane == 0)
            for (int w = 0; w < 8; w++) {   // end marker for every shard
                const int i = issued + ((w - issued) & 7);   // the next block number of shard w
                int st;
                uint32_t ph;
                slot(i, st, ph);
                if (i >= NST) mbar_wait(&empty[st], ph ^ 1);
                meta[st] = make_int4(-1, 0, 0, 0);
                mbar_arrive(&full[st]);
            }
        return;
    }
    // ----------------------------------------------------------------- consumers
    // the 256 consumer threads form ||x|| in k_norm_apply's order (256 strided partial sums,
    // then the halving tree; consumer-only named barrier) while the producer's first copies fly
    double nrm = 1.0;
    if (nrm_part) {
        double t = 0.0;
        for (int i = tid; i < np; i += 256) t += nrm_part[i];
        red[tid] = t;
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        for (int k = 128; k > 0; k >>= 1) {
            if (tid < k) red[tid] += red[tid + k];
            asm volatile("bar.sync 1, 256;\n" ::: "memory");
        }
        nrm = sqrt(red[0]);
    }
    double *vJ = vbuf + warp * 2 * B, *vI = vJ + B;
    for (int k = 0;; k++) {
        const int st = warp * BRS + k % BRS;
        mbar_wait(&full[st], (uint32_t)((k / BRS) & 1));
        const int4 mt = meta[st];
        if (mt.x < 0) break;
        const double *tile = sm + st * SD;
        const bool colpass = SYM && mt.z != mt.y;   // warp-uniform
        if (lane < B) {
            const double xj = SPAMM_SPB_VTMA ? tile[TILE + lane] : __ldg(g.v + (int64_t)mt.z * B + lane);
            vJ[lane] = nrm_part ? xj / nrm : xj;
            if (colpass) {
                const double xi = SPAMM_SPB_VTMA ? tile[TILE + B + lane] : __ldg(g.v + (int64_t)mt.y * B + lane);
                vI[lane] = nrm_part ? xi / nrm : xi;
            }
        }
        __syncwarp();
        if (lane < B) {
            double t = 0.0;
#pragma unroll
            for (int c = 0; c < B; c++) t = fma(tile[pool_at(lane, c, B)], vJ[c], t);
            bpart[(int64_t)mt.x * B + lane] = t;
            if (colpass) {
                double u = 0.0;
#pragma unroll
                for (int r = 0; r < B; r++) u = fma(tile[pool_at(r, lane, B)], vI[r], u);
                bpart[(int64_t)mt.w * B + lane] = u;
            }
        }
        // generic-proxy reads of the stage (and of vJ / vI) before its refill
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
}

// w[J*b + c] = sum over the CSR positions p of row J, ascending, of bpart[p*b + c]: SL = 256/b
// lanes per element each sum every SL-th position in order, then a fixed pairwise tree
// (deterministic); also the CTA's ||w||^2 partial (threads 0..b-1 hold the row: the reduction
// of k_row_sumsq).
template <int B>
__global__ void __launch_bounds__(256) k_spmv_bfix(const int32_t *rowptr, const double *bpart, double *w,
                                                   double *nrm_part)
{
    pdl_wait();
    pdl_trigger();
    constexpr int SL = 256 / B;
    __shared__ double sp[SL][B];
    const int J = blockIdx.x, c = threadIdx.x % B, q = threadIdx.x / B;
    const int p1 = rowptr[J + 1];
    double sl = 0.0;
    // loads in batches of 8 (independent of the running sum), then added in order
    for (int p0 = rowptr[J] + q; p0 < p1; p0 += 8 * SL) {
        double x[8];
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = p0 + i * SL < p1 ? bpart[(int64_t)(p0 + i * SL) * B + c] : 0.0;
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (p0 + i * SL < p1) sl += x[i];
    }
    sp[q][c] = sl;
    __syncthreads();
    double t = 0.0;
    if (q == 0) {
        double u[SL];
#pragma unroll
        for (int i = 0; i < SL; i++) u[i] = sp[i][c];
#pragma unroll
        for (int h = SL / 2; h > 0; h >>= 1)
#pragma unroll
            for (int i = 0; i < h; i++) u[i] += u[i + h];
        t = u[0];
        w[(int64_t)J * B + c] = t;
    }
    cta_sumsq_part(t, nrm_part);
}

// w[J*b + c] = (P0 + P1) + (P2 + P3) over J's upper quarters, then + the column
// parts of the blocks (I, J), I < J: colpart rows [rowptr[J], up[J]), ascending I.
// One CTA per block row J: SL = 256/b lanes per output element each sum every SL-th
// column part in order, and the lane partials join in a fixed pairwise tree
// (deterministic).  Also the CTA's partial of ||w||^2 (fused normalisation, k_norm_apply).
template <int B>
__global__ void __launch_bounds__(256) k_spmv_sym_fix(const int32_t *rowptr, const int32_t *up,
                                                      const double *part, const double *colpart,
                                                      double *w, double *nrm_part)
{
    pdl_wait();
    pdl_trigger();
    constexpr int SL = 256 / B;
    __shared__ double sp[SL][B];
    const int J = blockIdx.x, c = threadIdx.x % B, q = threadIdx.x / B;
    const int p0 = up[J];
    double sl = 0.0;
    for (int p = rowptr[J] + q; p < p0; p += SL) sl += colpart[(int64_t)p * B + c];
    sp[q][c] = sl;
    __syncthreads();
    double t = 0.0;
    if (q == 0) {
        const int len = rowptr[J + 1] - p0;
        double P[SPT_Q];
#pragma unroll
        for (int k = 0; k < SPT_Q; k++) {
            const bool any = ((k + 1) * len) / SPT_Q > (k * len) / SPT_Q;
            P[k] = any ? part[((int64_t)J * SPT_Q + k) * B + c] : 0.0;
        }
        double u[SL];
#pragma unroll
        for (int i = 0; i < SL; i++) u[i] = sp[i][c];
#pragma unroll
        for (int h = SL / 2; h > 0; h >>= 1)
#pragma unroll
            for (int i = 0; i < h; i++) u[i] += u[i + h];
        t = ((P[0] + P[1]) + (P[2] + P[3])) + u[0];
        w[(int64_t)J * B + c] = t;
    }
    cta_sumsq_part(t, nrm_part);
}

// Structure of the symmetric SpMV, one CTA per block row J:
//   up[J]   = first CSR position of row J with column >= J;
//   mir[p]  = CSR position of the mirror (I, J) of the entry p = (J, I) (p itself on
//             the diagonal).
// *bad = 1 if some block has no mirror (the pattern is not symmetric).
__global__ void k_sym_index(const int32_t *rowptr, const int32_t *cols, int nb, int32_t *up,
                            int32_t *mir, int32_t *bad)
{
    const int J = blockIdx.x, p0 = rowptr[J], p1 = rowptr[J + 1];
    if (threadIdx.x == 0 && (p1 == p0 || cols[p0] >= J)) up[J] = p0;
    for (int p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const int I = cols[p];
        if (I < J && (p + 1 == p1 || cols[p + 1] >= J)) up[J] = p + 1;
        if (I == J) {
            mir[p] = p;
            continue;
        }
        int lo = rowptr[I], hi = rowptr[I + 1];   // binary search for J in row I
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cols[mid] < J) lo = mid + 1;
            else hi = mid;
        }
        const bool found = lo < rowptr[I + 1] && cols[lo] == J;
        if (!found) *bad = 1;
        else mir[p] = lo;
    }
}

// *bad = 1 unless S_JI == S_IJ^T bitwise for every block on or below the diagonal
// (one CTA per CSR position; positions above the diagonal return at once)
template <int B>
__global__ void __launch_bounds__(256) k_sym_check(const double *pool, const int32_t *rowptr,
                                                   const int32_t *cols, const int32_t *slots,
                                                   const int32_t *mir, int nb, int32_t *bad)
{
    __shared__ double t[B * B];
    const int p = blockIdx.x;
    int lo = 0, hi = nb;   // row of p: last J with rowptr[J] <= p
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (rowptr[mid] <= p) lo = mid;
        else hi = mid;
    }
    const int J = lo, I = cols[p];
    if (I > J || *(volatile int32_t *)bad) return;   // upper entry, or k_sym_index found no mirror
    const int q = mir[p];
    const double *a = pool + (int64_t)slots[p] * B * B, *m = pool + (int64_t)slots[q] * B * B;
    for (int e = threadIdx.x; e < B * B; e += 256) t[e] = m[e];
    __syncthreads();
    bool ok = true;
    for (int e = threadIdx.x; e < B * B; e += 256) {
        const int r = e / B, c = pool_col(e, B);
        ok &= __double_as_longlong(a[e]) == __double_as_longlong(t[pool_at(c, r, B)]);
    }
    if (__syncthreads_or(!ok) && threadIdx.x == 0) *bad = 1;
}

// v = w / sqrt(sum of the np partials); every CTA sums the partials in the same fixed
// order (strided per thread, then a tree), so all agree bitwise on the norm
__global__ void __launch_bounds__(256) k_norm_apply(const double *w, int64_t n, const double *nrm_part, int np,
                                                    double *v)
{
    pdl_wait();
    pdl_trigger();
    __shared__ double sh[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += 256) s += nrm_part[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
        __syncthreads();
    }
    const double nrm = sqrt(sh[0]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = w[i] / nrm;
}

// single CTA: nrm = sqrt(sum w^2) (fixed order); v = w / nrm
__global__ void k_normalize(const double *w, int64_t n, double *v)
{
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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

struct SymSpmv {
    const int32_t *up, *mir;   // mir only for SYM
    double *colpart;
};

// w = s v with the TMA kernel.  SYM: the upper block triangle only (s symmetric);
// otherwise the upper parts plus the lower blocks' column parts, which for a symmetric
// s are bit for bit the SYM kernel's, so both (and the row-partitioned path) give the
// same w.  Then the fix-up: w rows and their ||w||^2 partials (one per block row).
template <int B, bool SYM>
static spamm_status spmv_tma(spamm_ctx ctx, spamm_mat s, const int32_t *rowptr, const int32_t *cols,
                             const int32_t *slots, const double *v, double *w, int32_t *ticket, double *part,
                             double *nrm_part, const SymSpmv &y, int rev)
{
    constexpr int STAGES = SptCfg<B>::STAGES;
    const size_t smem = sizeof(double) * STAGES * B * B + STAGES * (2 * sizeof(uint64_t) + sizeof(int4));
    static std::atomic<uint64_t> configured{0};
    CK(once_per_device(configured, ctx->device, [&]() {
        return cudaFuncSetAttribute(k_spmv_tma<B, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }));
    const int nupper = s->nb * SPT_Q;
    SpmvTmaArgs g{s->pool, rowptr, cols, slots, v, part, ticket, nupper, SYM ? nupper : nupper + s->nb, rev};
    if (s->dist) {   // the predecessor is a collective: plain launches
        k_spmv_tma<B, SYM><<<ctx->sm_count, 288, smem, ctx->stream>>>(g, y.up, y.mir, y.colpart);
        CKL(ctx);
        k_spmv_sym_fix<B><<<s->nb, 256, 0, ctx->stream>>>(rowptr, y.up, part, y.colpart, w, nrm_part);
    } else {
        CK(launch_pdl(k_spmv_tma<B, SYM>, ctx->sm_count, 288, smem, ctx->stream, g, y.up, y.mir, y.colpart));
        CKL(ctx);
        CK(launch_pdl(k_spmv_sym_fix<B>, s->nb, 256, 0, ctx->stream, rowptr, y.up, (const double *)part,
                      (const double *)y.colpart, w, nrm_part));
    }
    CKL(ctx);
    return SPAMM_OK;
}

// w = s v with the per-block kernel (b = 32 / 16), then the fix-up: w rows and their ||w||^2
// partials (one per block row).  bpart: one b-vector per CSR position.
// xnrm (nullable): v is x / ||x|| with ||x||^2 = the sum of xnrm's nb partials (fused
// normalisation, single device)
template <int B, bool SYM>
static spamm_status spmv_blk(spamm_ctx ctx, spamm_mat s, const int32_t *rowptr, const int32_t *cols,
                             const int32_t *slots, const double *v, double *w, int32_t *ticket,
                             double *nrm_part, const SymSpmv &y, int rev, const double *xnrm)
{
    const size_t smem = SpbCfg<B>::smem;
    static std::atomic<uint64_t> configured{0};
    CK(once_per_device(configured, ctx->device, [&]() {
        return cudaFuncSetAttribute(k_spmv_blk<B, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }));
    const int nunits = s->nb * SPT_Q;
    SpmvTmaArgs g{s->pool, rowptr, cols, slots, v, nullptr, ticket, nunits, nunits, rev};
    if (s->dist) {   // the predecessor is a collective: plain launches
        k_spmv_blk<B, SYM><<<ctx->sm_count, 288, smem, ctx->stream>>>(g, y.up, y.mir, y.colpart, nullptr, 0);
        CKL(ctx);
        k_spmv_bfix<B><<<s->nb, 256, 0, ctx->stream>>>(rowptr, y.colpart, w, nrm_part);
    } else {
        CK(launch_pdl(k_spmv_blk<B, SYM>, ctx->sm_count, 288, smem, ctx->stream, g, y.up, y.mir, y.colpart, xnrm,
                      s->nb));
        CKL(ctx);
        CK(launch_pdl(k_spmv_bfix<B>, s->nb, 256, 0, ctx->stream, rowptr, (const double *)y.colpart, w, nrm_part));
    }
    CKL(ctx);
    return SPAMM_OK;
}

// ||w||^2 partials per block row of the gathered w (row partition), with exactly the
// reduction of k_spmv_sym_fix (threads 0..b-1 hold the row's entries)
template <int B>
__global__ void __launch_bounds__(256) k_row_sumsq(const double *w, double *nrm_part)
{
    pdl_wait();
    pdl_trigger();
    const double t = threadIdx.x < B ? w[(int64_t)blockIdx.x * B + threadIdx.x] : 0.0;
    cta_sumsq_part(t, nrm_part);
}

template <int B>
static spamm_status spmv(spamm_ctx ctx, spamm_mat s, const int32_t *rowptr, const int32_t *cols,
                         const int32_t *slots, const double *v, double *w, int32_t *ticket, int rev)
{
    // NT = 64: more, smaller units than 256 threads (C2 setup 3.37 -> 3.23 ms, C1 0.74 ->
    // 0.66 ms); the register-light 64-thread CTAs also fill the SMs better
    constexpr int NT = 64;
    constexpr int E = B >= 32 ? 4 : 1, TPR = B / E, RG = NT / TPR, CPR = B / RG;
    static std::atomic<int> occ_cache{0};
    int occ = occ_cache.load();
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv<B, NT>, NT, 0);
        if (occ < 1) occ = 1;
        occ_cache.store(occ);
    }
    const int nunits = s->nb * CPR;
    int grid = ctx->sm_count * occ;
    if (grid > nunits) grid = nunits;
    if (s->dist) k_spmv<B, NT><<<grid, NT, 0, ctx->stream>>>(s->pool, rowptr, cols, slots, v, w, ticket, nunits, rev);
    else CK(launch_pdl(k_spmv<B, NT>, grid, NT, 0, ctx->stream, s->pool, rowptr, cols, slots, v, w, ticket, nunits, rev));
    CKL(ctx);
    return SPAMM_OK;
}

// ------------------------------------------------- tiny s: the whole iteration on one cluster
// For the smallest problems (C1: n = 256, 512 KB of blocks) every launch of the power
// iteration is latency: 2 launches per step, ~6.4 us.  Here a cluster of PC_CN CTAs keeps s
// resident in shared memory for all K + 1 SpMVs (CTA q owns the block rows I = q mod PC_CN)
// and exchanges w through distributed shared memory, one cluster barrier per step.  The
// arithmetic is exactly that of the launch loop it replaces (k_spmv: per lane, E-term fma
// chains added to acc over the row's blocks in CSR order, then the TPR lanes' xor tree;
// k_normalize: 1024 fma partials and its halving tree; k_dot likewise), so c is bitwise the
// same (tests/test_gpu_parity.py::test_power_cluster_bitwise).
constexpr int PC_CN = 8;     // CTAs per cluster (portable size)
constexpr int PC_NT = 256;   // threads per CTA

template <int B>
__global__ void __launch_bounds__(PC_NT) k_power_cluster(const double *pool, const int32_t *rowptr,
                                                         const int32_t *cols, const int32_t *slots, int nb,
                                                         int K, double v0, double *c_out)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int E = B >= 32 ? 4 : 1, TPR = B / E;
    const int q = (int)cl.block_rank();
    const int n = nb * B;
    extern __shared__ __align__(16) double pc_smem[];
    double *red = pc_smem;                 // [1024] reduction slots
    double *v = red + 1024;                // [n]
    double *wb[2] = {v + n, v + 2 * n};    // [n] each: w, written by every CTA of the cluster
    double *sb = v + 3 * n;                // this CTA's blocks, its rows in order, CSR order inside
    // stage the blocks of the owned rows
    int nloc = 0;
    for (int I = q; I < nb; I += PC_CN) {
        const int p0 = rowptr[I], p1 = rowptr[I + 1];
        for (int p = p0; p < p1; p++) {
            const double *src = pool + (int64_t)slots[p] * B * B;
            double *dst = sb + (int64_t)(nloc + p - p0) * B * B;
            for (int e = threadIdx.x; e < B * B; e += PC_NT) dst[e] = src[e];
        }
        nloc += p1 - p0;
    }
    for (int i = threadIdx.x; i < n; i += PC_NT) v[i] = v0;
    const int nown = (nb - q + PC_CN - 1) / PC_CN;
    const int items = nown * B * TPR;   // (row, lane) pairs: a multiple of 32
    __syncthreads();
    for (int it = 0; it <= K; it++) {
        double *w = wb[it & 1];
        // w rows of the owned block rows: k_spmv's per-lane arithmetic and xor tree
        for (int base = 0; base < items; base += PC_NT) {
            const int x = base + threadIdx.x;
            double acc = 0.0;
            int I = 0, r = 0;
            if (x < items) {
                const int lrow = x / TPR, t = x % TPR;
                const int li = lrow / B;
                r = lrow % B;
                I = q + li * PC_CN;
                // local block index of row I's first block: the rows before it, in order
                int lb = 0;
                for (int J = q; J < I; J += PC_CN) lb += rowptr[J + 1] - rowptr[J];
                const int p0 = rowptr[I], p1 = rowptr[I + 1];
                const int e0 = r * B + t * E;
                int lc[E];
#pragma unroll
                for (int i = 0; i < E; i++) lc[i] = pool_col(e0 + i, B);
                for (int p = p0; p < p1; p++) {
                    const double *blk = sb + (int64_t)(lb + p - p0) * B * B + e0;
                    const double *vv = v + (int64_t)cols[p] * B;
                    double sdot = 0.0;
#pragma unroll
                    for (int i = 0; i < E; i++) sdot = fma(blk[i], vv[lc[i]], sdot);
                    acc += sdot;
                }
            }
#pragma unroll
            for (int o = 1; o < TPR; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (x < items && (x % TPR) == 0) {
                const int gi = I * B + r;
                for (int d = 0; d < PC_CN; d++) cl.map_shared_rank(w, d)[gi] = acc;
            }
        }
        cl.sync();   // every w row has landed in every CTA (release / acquire)
        // it < K: v = w / ||w|| (k_normalize); it == K: c = v . w (k_dot)
        for (int t = threadIdx.x; t < 1024; t += PC_NT) {
            double a = 0.0;
            for (int i = t; i < n; i += 1024) a = it < K ? fma(w[i], w[i], a) : fma(v[i], w[i], a);
            red[t] = a;
        }
        __syncthreads();
        for (int k = 512; k > 0; k >>= 1) {
            for (int t = threadIdx.x; t < k; t += PC_NT) red[t] += red[t + k];
            __syncthreads();
        }
        if (it < K) {
            const double nrm = sqrt(red[0]);
            for (int i = threadIdx.x; i < n; i += PC_NT) v[i] = w[i] / nrm;
            __syncthreads();
        } else if (q == 0 && threadIdx.x == 0) {
            *c_out = red[0];
        }
    }
}

// bytes of shared memory k_power_cluster<B> needs for s in the worst case (dense rows), or
// 0 if it is not eligible
static size_t power_cluster_smem(const spamm_mat s)
{
    const int64_t nb = s->nb, n = s->n, b = s->b;
    const int64_t rows = (nb + PC_CN - 1) / PC_CN;
    const int64_t bytes = sizeof(double) * (1024 + 3 * n + rows * nb * b * b);
    return bytes <= 200 * 1024 ? (size_t)bytes : 0;
}

// SPAMM_POWER_CLUSTER=0: the launch loop even where the cluster kernel fits (A/B, tests)
static bool power_cluster_mode()
{
    static const int m = [] {
        const char *e = getenv("SPAMM_POWER_CLUSTER");
        return e && *e ? atoi(e) : 1;
    }();
    return m != 0;
}

template <int B>
static spamm_status power_cluster(spamm_ctx ctx, spamm_mat s, const int32_t *rowptr, const int32_t *cols,
                                  const int32_t *slots, int K, double v0, double *c, size_t smem)
{
    static std::atomic<uint64_t> configured{0};
    CK(once_per_device(configured, ctx->device, [&]() {
        return cudaFuncSetAttribute(k_power_cluster<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(PC_CN);
    cfg.blockDim = dim3(PC_NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PC_CN;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_power_cluster<B>, s->pool, rowptr, cols, slots, (int)s->nb, K, v0, c));
    ctx->launches++;
    CKL(ctx);
    return SPAMM_OK;
}

// SPAMM_SPMV_TMA=0 selects the register-streaming SpMV (k_spmv) instead of the TMA
// ring; SPAMM_SPMV_SYM=0 disables the symmetric (upper-half) SpMV
// 0 = off, 1 = b = 64 (default), 2 = every leaf size (measurement)
static int spmv_tma_mode()
{
    static const int m = [] {   // function-local static: thread-safe init
        const char *e = getenv("SPAMM_SPMV_TMA");
        return e && *e ? atoi(e) : 1;
    }();
    return m;
}
// SPAMM_SPMV_BLK: 0 = the register-streaming SpMV for b = 32 too, 1 = per-block kernel for
// b = 32 (default), 2 = also for b = 16 (A/B runs)
static int spmv_blk_mode()
{
    static const int m = [] {
        const char *e = getenv("SPAMM_SPMV_BLK");
        return e && *e ? atoi(e) : 1;
    }();
    return m;
}
// 0 = off, 1 = b = 64 (default), 2 = every leaf size (measurement)
static int spmv_sym_mode()
{
    static const int m = [] {
        const char *e = getenv("SPAMM_SPMV_SYM");
        return e && *e ? atoi(e) : 1;
    }();
    return m;
}

// SPAMM_SPMV_ZIGZAG=0: every SpMV takes its units in ascending order (A/B runs)
static int zigzag_mode()
{
    static const int m = [] {
        const char *e = getenv("SPAMM_SPMV_ZIGZAG");
        return e && *e ? atoi(e) : 1;
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
    const int tmam = spmv_tma_mode();
    const bool tma = tmam == 2 || (tmam == 1 && s->b == 64);
    // b = 32 / 16: the per-block kernel (one warp per block, results per block, no CTA barrier)
    // (b = 16 keeps the register kernel: C1, n = 256, is launch-bound and the fix-up launch
    // costs more than it saves: 0.67 vs 0.98 ms per power iteration)
    const bool blk = !tma && (s->b == 32 || (s->b == 16 && spmv_blk_mode() == 2)) && spmv_blk_mode() != 0;
    const bool ring = tma || blk;   // fix-up + fused normalisation; symmetric read possible
    // symmetric s (checked below, single device): read only the upper half of the blocks
    const int symm = spmv_sym_mode();
    bool sym = ring && !s->dist && (symm == 2 || (symm == 1 && (s->b == 64 || blk)));
    double *part = tma ? dalloc<double>(ctx, (int64_t)nb * SPT_Q * s->b) : nullptr;
    double *nrm_part = ring ? dalloc<double>(ctx, nb) : nullptr;   // ||w||^2 partials, one per block row
    int32_t *up = ring ? dalloc<int32_t>(ctx, nb) : nullptr, *mir = ring ? dalloc<int32_t>(ctx, nblk) : nullptr;
    // column parts (TMA ring) / per-block parts (per-block kernel), one b-vector per CSR position
    double *colpart = ring ? dalloc<double>(ctx, nblk * s->b) : nullptr;
    // every exit (errors included) goes through the one cleanup below
    auto body = [&]() -> spamm_status {
    if (!cnt || !rowptr || !cols || !slots || !v || !w || !c || !tickets || (tma && !part) ||
        (ring && (!nrm_part || !up || !mir || !colpart)))
        return set_err(ctx, SPAMM_ENOMEM, "power");
    CK(cudaMemsetAsync(tickets, 0, sizeof(int32_t) * (K + 1), ctx->stream));
    int nmv = 0;
    cudaStream_t st = ctx->stream;
    k_row_count<<<nb, 256, 0, st>>>(s->slot, nb, cnt);
    k_row_scan<<<1, 1024, 0, st>>>(cnt, nb, rowptr);
    k_row_fill<<<nb, 256, 0, st>>>(s->slot, nb, rowptr, cols, slots);
    k_fill<<<cdiv(n, 256), 256, 0, st>>>(v, n, 1.0 / sqrt((double)n));
    ctx->launches += 4;
    SymSpmv sy{up, mir, colpart};
    if (ring) {
        // up[] for every TMA SpMV; the mirror positions and the bitwise symmetry check
        // only where the symmetric kernel may run (with a row partition some mirrors
        // live on other ranks)
        int32_t *bad = reinterpret_cast<int32_t *>(c);   // c[0] is written only by the final dot
        CK(cudaMemsetAsync(bad, 0, sizeof(int32_t), st));
        k_sym_index<<<nb, 256, 0, st>>>(rowptr, cols, nb, up, mir, bad);
        ctx->launches++;
        if (sym && s->nblk > 0) {
            switch (s->b) {
            case 16: k_sym_check<16><<<(int)s->nblk, 256, 0, st>>>(s->pool, rowptr, cols, slots, mir, nb, bad); break;
            case 32: k_sym_check<32><<<(int)s->nblk, 256, 0, st>>>(s->pool, rowptr, cols, slots, mir, nb, bad); break;
            default: k_sym_check<64><<<(int)s->nblk, 256, 0, st>>>(s->pool, rowptr, cols, slots, mir, nb, bad); break;
            }
            ctx->launches++;
        }
        CKL(ctx);
        if (sym) {
            int32_t hbad = 1;
            ST(fetch1(ctx, bad, &hbad, sizeof(int32_t)));
            sym = hbad == 0;
        }
    }
    // row partition: local block rows of w = s v, then all ranks gather the full w and
    // form the norm partials from it (each row is computed by one rank with the
    // single-device arithmetic: bitwise G-invariant)
    // Zig-zag: consecutive SpMVs take their work units in opposite orders, so each pass
    // starts on the blocks the previous one touched last, which are still in L2 (s of
    // C2 is 132 MB, the symmetric half of C3's 165 MB: around the 126 MB of L2).  Only
    // the schedule changes; every row is summed in the same order: w is bitwise the same.
    auto mv = [&](const double *x, double *y, int32_t *tk, const double *xnrm = nullptr) -> spamm_status {
        const int rev = zigzag_mode() ? (int)((tk - tickets) & 1) : 0;
        if (ring) {
            if (blk) {
                spamm_status r = s->b == 32
                    ? (sym ? spmv_blk<32, true>(ctx, s, rowptr, cols, slots, x, y, tk, nrm_part, sy, rev, xnrm)
                           : spmv_blk<32, false>(ctx, s, rowptr, cols, slots, x, y, tk, nrm_part, sy, rev, xnrm))
                    : (sym ? spmv_blk<16, true>(ctx, s, rowptr, cols, slots, x, y, tk, nrm_part, sy, rev, xnrm)
                           : spmv_blk<16, false>(ctx, s, rowptr, cols, slots, x, y, tk, nrm_part, sy, rev, xnrm));
                ST(r);
            } else switch (s->b) {
            case 16: {
                spamm_status r = sym ? spmv_tma<16, true>(ctx, s, rowptr, cols, slots, x, y, tk, part, nrm_part, sy, rev)
                                     : spmv_tma<16, false>(ctx, s, rowptr, cols, slots, x, y, tk, part, nrm_part, sy, rev);
                ST(r);
                break;
            }
            case 32: {
                spamm_status r = sym ? spmv_tma<32, true>(ctx, s, rowptr, cols, slots, x, y, tk, part, nrm_part, sy, rev)
                                     : spmv_tma<32, false>(ctx, s, rowptr, cols, slots, x, y, tk, part, nrm_part, sy, rev);
                ST(r);
                break;
            }
            default: {
                spamm_status r = sym ? spmv_tma<64, true>(ctx, s, rowptr, cols, slots, x, y, tk, part, nrm_part, sy, rev)
                                     : spmv_tma<64, false>(ctx, s, rowptr, cols, slots, x, y, tk, part, nrm_part, sy, rev);
                ST(r);
                break;
            }
            }
            if (s->dist) {
                ST(gather_rows(ctx, s->parts, y, s->b));
                switch (s->b) {
                case 16: k_row_sumsq<16><<<nb, 256, 0, st>>>(y, nrm_part); break;
                case 32: k_row_sumsq<32><<<nb, 256, 0, st>>>(y, nrm_part); break;
                default: k_row_sumsq<64><<<nb, 256, 0, st>>>(y, nrm_part); break;
                }
                CKL(ctx);
            }
            return SPAMM_OK;
        }
        switch (s->b) {
        case 16: ST(spmv<16>(ctx, s, rowptr, cols, slots, x, y, tk, rev)); break;
        case 32: ST(spmv<32>(ctx, s, rowptr, cols, slots, x, y, tk, rev)); break;
        default: ST(spmv<64>(ctx, s, rowptr, cols, slots, x, y, tk, rev)); break;
        }
        return s->dist ? gather_rows(ctx, s->parts, y, s->b) : SPAMM_OK;
    };
    // one power step: w = s v, then v = w / ||w|| (its ticket zeroed first)
    auto power_step = [&](int32_t *tk) -> spamm_status {
        ST(mv(v, w, tk));
        if (ring) {   // the fix-up's (or, row partition, k_row_sumsq's) per-block-row partials
            const int g = (int)std::min<int64_t>(NRM_CTAS, nb);
            if (s->dist) k_norm_apply<<<g, 256, 0, st>>>(w, n, nrm_part, nb, v);
            else CK(launch_pdl(k_norm_apply, g, 256, 0, st, (const double *)w, n, (const double *)nrm_part, nb, v));
        } else if (n >= (1 << 16)) {
            k_sumsq_part<<<NRM_CTAS, 256, 0, st>>>(w, n, c + 1);
            k_scale_by_norm<<<NRM_CTAS, 256, 0, st>>>(w, n, c + 1, v);
            ctx->launches++;
        } else {
            if (s->dist) k_normalize<<<1, 1024, 0, st>>>(w, n, v);
            else CK(launch_pdl(k_normalize, 1, 1024, 0, st, (const double *)w, n, v));
        }
        ctx->launches++;
        return SPAMM_OK;
    };
    const size_t pcs = (!ring && !s->dist && K > 0 && (s->b == 16 || s->b == 32) && power_cluster_mode())
                           ? power_cluster_smem(s) : 0;
    if (pcs) {
        // tiny s: the whole iteration (v0 as k_fill's) on one cluster, s resident in shared memory
        const double v0 = 1.0 / sqrt((double)n);
        ST(s->b == 16 ? power_cluster<16>(ctx, s, rowptr, cols, slots, K, v0, c, pcs)
                      : power_cluster<32>(ctx, s, rowptr, cols, slots, K, v0, c, pcs));
    } else if (blk && !s->dist && K > 0) {
        // per-block kernel on one device: v <- w / ||w|| is folded into the next SpMV (every CTA
        // forms ||w|| from the fix-up's partials in k_norm_apply's order), so a power step is
        // two launches; w and v alternate as the SpMV's input and output
        double *x = v, *y = w;
        const double *xn = nullptr;
        for (int it = 0; it < K; it++) {
            ST(mv(x, y, tickets + nmv++, xn));
            xn = nrm_part;
            std::swap(x, y);   // x = w_it
        }
        // materialise v_K = w_K / ||w_K||, then w = s v_K and c = v_K . w
        const int g = (int)std::min<int64_t>(NRM_CTAS, nb);
        CK(launch_pdl(k_norm_apply, g, 256, 0, st, (const double *)x, n, (const double *)nrm_part, nb, y));
        ctx->launches++;
        ST(mv(y, x, tickets + K));
        k_dot<<<1, 1024, 0, st>>>(y, x, n, c);
    } else {
        for (int it = 0; it < K; it++) ST(power_step(tickets + nmv++));
        ST(mv(v, w, tickets + K));
        k_dot<<<1, 1024, 0, st>>>(v, w, n, c);
    }
    CKL(ctx);
    double h = 0;
    ST(fetch1(ctx, c, &h, sizeof(double)));
    *c_host = h;
    return SPAMM_OK;
    };
    const spamm_status result = body();
    dev_free(ctx, cnt, sizeof(int32_t) * nb);
    dev_free(ctx, rowptr, sizeof(int32_t) * (nb + 1));
    dev_free(ctx, cols, sizeof(int32_t) * nblk);
    dev_free(ctx, slots, sizeof(int32_t) * nblk);
    dev_free(ctx, v, sizeof(double) * n);
    dev_free(ctx, w, sizeof(double) * n);
    dev_free(ctx, c, sizeof(double) * (1 + NRM_CTAS));
    dev_free(ctx, tickets, sizeof(int32_t) * (K + 1));
    dev_free(ctx, part, sizeof(double) * (int64_t)nb * SPT_Q * s->b);
    dev_free(ctx, nrm_part, sizeof(double) * nb);
    dev_free(ctx, up, sizeof(int32_t) * nb);
    dev_free(ctx, mir, sizeof(int32_t) * nblk);
    dev_free(ctx, colpart, sizeof(double) * nblk * s->b);
    return result;
}
