// gemm.cu — the batched leaf-block GEMM of SpAMM on FP64 tensor cores (sm_100a).
//
// For every output segment (i,j) produced by the cull (tasks sorted by k):
//     C_ij = sum_{k in S_ij} A_ik . B_kj            (Eq. newspamm leaf)
// accumulated in registers in ascending k (segmented in-register reduction, no
// atomics), with fused epilogues:
//   EPI_STORE : C_ij -> pool, ||C_ij||^2 -> leaf level of the norm pyramid
//   EPI_NS_H  : H_ij = 1/2 (3 delta_ij I - X_ij) (alpha = 1) -> pool,
//               ||H_ij||^2, and tr(X_ii) partials for t_k;
//               X itself is never stored.
//   EPI_NS_X  : X_ij -> pool, ||X_ij||^2, tr(X_ii) partials (scaled map: the
//               coefficients alpha(t_k), eps(t_k) need the full trace first, so
//               k_ns_map applies H = h_alpha[(1-2eps)X + eps I] in a second pass).
// FP64 MMA on sm_100a is warp-level mma.sync m8n8k4 (SASS DMMA.8x8x4); tcgen05
// has no f64 kind, so operands go shared memory -> registers.  Tiles are staged
// by a warp-specialised TMA bulk-copy / mbarrier pipeline; the pool layout is
// pre-swizzled (common.cuh pool_at) so both fragment patterns are conflict-free:
//   A: lane (g,t) reads A[g][4t..4t+3] (2 x LDS.128) — the contraction index is
//      permuted inside each 16-wide k chunk as k = 4t + s (same permutation on
//      B's rows, so the product is unchanged);
//   B: lane (g,t) reads B[4t+s][g] (LDS.64).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "scan.cuh"
#include "tma.cuh"

// EPI_STORE with alpha != 1 (C = alpha (A (x) B)): a separate instance, so the plain
// store epilogue carries no multiply
constexpr int EPI_STORE_SCALED = 3;

struct GemmArgs {
    const double *a_pool, *b_pool;
    const double *b_halo;   // remote right-operand tiles (row partition): tB = -(h+1)
    const int32_t *tA, *tB;
    const int32_t *seg_code, *seg_start, *seg_len;
    int nseg;               // segments of this launch
    const int32_t *seg_order;  // nullable: launch-local ticket q -> segment seg_order[q]
    double *c_pool;
    int32_t *c_coord, *c_slot;
    double *c_leaf_n2;
    double *trace_part;
    int32_t *ticket;   // dynamic segment scheduler (zeroed before the launch)
    double alpha;      // EPI_STORE: C = alpha (A (x) B) (the final unscale of the NS run, fused)
    const int32_t *nseg_dev;   // non-null: the segment count is read here (device-driven
                               // steps: the cull's count, no host round trip)
    int peer_world;            // > 0: tB < 0 is -(slot * peer_world + owner) - 1, a tile read in
    const double *peer_pool[SPAMM_MAX_WORLD];   // place from the owner's pool (peer memory)
    // capacities, checked by the SPAMM_DEBUG build only
    int64_t a_cap, b_cap, halo_cap, c_cap, task_cap, seg_cap;
    int nb;
};

#ifdef SPAMM_GEMM_CLOCKS
// diagnostic build only (tools/gemm_clocks.py): consumer-warp cycle accounting
// [0] loop total, [1] waiting for a stage (full), [2] waiting for a queue entry,
// [3] segment boundaries (map, partials, deposit), [4] tasks, [5] segments, [6] of [3]: the
// map and partials, [7] of [3]: waiting for the epilogue warp to release the tile
__device__ unsigned long long g_gemm_clk[8];
extern "C" int spamm_debug_gemm_clocks(unsigned long long *out, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_gemm_clk, sizeof(g_gemm_clk));
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(g_gemm_clk, z, sizeof(z));
    }
    return (int)cudaDeviceSynchronize();
}
#define CLK(...) __VA_ARGS__
#else
#define CLK(...)
#endif

__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Warp-specialised persistent leaf GEMM.
//   warp CW (producer): one elected lane takes segments from a global ticket
//     (dynamic scheduling, Morton order: no tail imbalance, deterministic
//     results since a segment is owned by one CTA), announces each through a
//     smem queue, and per task waits for a free stage, then TMA-bulk-copies the
//     A and B tiles (b*b*8 bytes each, pre-swizzled in the pool) into it.
//   warps 0..CW-1 (consumers): per task wait for the stage, load fragments,
//     issue DMMAs into register accumulators, release the stage; at the end of a
//     segment apply the value map (H = 1.5 delta - 0.5 X, alpha), form their share
//     of ||C_ij||^2 (and tr X_ii) in short FMA chains, deposit values (eswz layout)
//     and partial in the smem epilogue tile and go on to the next segment.
//   warps CW+1 .. CW+EW (epilogue): copy the deposited tile to the pool with
//     contiguous 16-byte stores; the first also sums the consumers' partials in a
//     fixed order (deterministic) and writes the block's metadata.
// The consumers issue no global stores, shuffle trees or cross-warp hand-offs, so
// the DMMA pipe keeps running across segment boundaries.  Measured on the C5 k = 8
// products (4.6 tasks per segment; tools/gemm_clocks.py): the whole epilogue in the
// consumer warps, interleaved with the next segment's first task, took 4.2 % of their
// cycles + 0.9 % at the boundary; here the boundary is ~3.8 %.  EW = 2 measured best
// (NS step GEMM 59.61 ms against 59.98 before, EW = 1: 59.65, EW = 4: 60.02); a single
// epilogue warp that also did the map and norms fell behind (the FP64 pipe is busy with
// DMMAs: 10.7 % of the consumers' cycles waiting for the tile), and a TMA bulk store of
// the tile needs a proxy fence in every consumer thread (5.6 % at the boundary).
// TA = 1: the left operand is A^T (single channel, §8(f) f2): the A tile is read
// with the column pattern of the B fragments (A^T[m][k] = A[k][m]).
// The epilogue tile's own chunk swizzle: chunk c/2 of row r at (c/2) ^ eswz(r).  A deposit
// instruction (rows 8mf + g8, chunks 4nf + t4 + const) then fills 8 distinct 16-byte bank
// slots in each 8-lane phase (the pool swizzle would put rows 2p and 2p+1 on the same 4:
// two-way conflicts); the epilogue warps read whole rows and store them in the pool layout.
__device__ __forceinline__ int eswz(int r) { return (r & 1) << 2; }

template <int B, int CW, int STAGES>
struct GemmSmem {
    static constexpr int TILE = B * B;
    static constexpr int QN = 4;   // segment-queue depth (producer -> consumers)
    // doubles: STAGES x {A, B} tiles, the epilogue tile, the consumers' per-lane ||.||^2
    // partials and per-warp trace partials; then the barriers, the queue and the record
    static constexpr int ETR = (CW + 1) & ~1;   // tr partials, padded to keep 16-byte alignment
    static constexpr size_t bytes = sizeof(double) * ((2 * STAGES + 1) * TILE + 32 * CW + ETR) +
                                    sizeof(uint64_t) * (2 * STAGES + 2 * QN + 2) + sizeof(int4) * (QN + 1);
    static_assert(bytes <= 227 * 1024, "the leaf GEMM's shared memory exceeds the 227 KiB an sm_100a CTA may use");
};

#ifndef SPAMM_EPI_WARPS
#define SPAMM_EPI_WARPS 2
#endif
constexpr int EW = SPAMM_EPI_WARPS;   // epilogue warps

template <int B, int CW, int WM, int WN, int STAGES, int EPI, int TA>
__global__ void __launch_bounds__(32 * (CW + 1 + EW), 1) k_leaf_gemm(GemmArgs g)
{
    static_assert(WM * WN == CW, "warp grid");
    constexpr bool STORE = EPI == EPI_STORE || EPI == EPI_STORE_SCALED;
    constexpr int TM = B / WM, TN = B / WN;
    constexpr int MF = TM / 8, NF = TN / 8;
    constexpr int TILE = B * B;
    constexpr uint32_t TILE_BYTES = TILE * 8;
    extern __shared__ __align__(1024) double smem[];
    constexpr int QN = GemmSmem<B, CW, STAGES>::QN;
    double *ebuf = smem + 2 * STAGES * TILE;                  // the epilogue tile (eswz layout)
    double *ess = ebuf + TILE;                                // [CW][32] lanes' ||C_ij||^2 partials
    double *etr = ess + 32 * CW;                              // [CW] warps' tr partials (diagonal blocks)
    uint64_t *full = reinterpret_cast<uint64_t *>(etr + GemmSmem<B, CW, STAGES>::ETR);
    uint64_t *empty = full + STAGES;
    uint64_t *qfull = empty + STAGES;
    uint64_t *qempty = qfull + QN;
    uint64_t *efull = qempty + QN;                            // tile deposited (CW arrivals)
    uint64_t *eempty = efull + 1;                             // tile stored by the epilogue warp
    int4 *segq = reinterpret_cast<int4 *>(eempty + 1);        // {seg, len, code, -} per queue entry
    int4 *erec = segq + QN;                                   // {seg, code} of the deposited tile

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_trigger();   // the epilogue-side kernels that follow may stage their launch now
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        for (int q = 0; q < QN; q++) {
            mbar_init(&qfull[q], 1);
            mbar_init(&qempty[q], CW);
        }
        mbar_init(efull, CW);
        mbar_init(eempty, EW);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == CW) {
        // ------------------------------------------------------- producer
        // Dynamic scheduling: segments (Morton order) are taken from a global
        // ticket and announced to the consumers through a QN-deep smem queue.
        int stage = 0, q = 0;
        uint32_t phase = 0, qphase = 0;
        for (;;) {
            int seg = 0, start = 0, len = 0;
            if (lane == 0) {
                seg = atomicAdd(g.ticket, 1);
                if (seg >= (g.nseg_dev ? *g.nseg_dev : g.nseg)) seg = -1;
                else if (g.seg_order) seg = g.seg_order[seg];
                int code = 0;
                if (seg >= 0) {
                    SPAMM_ASSERT(seg < g.seg_cap);
                    start = g.seg_start[seg];
                    len = g.seg_len[seg];
                    code = g.seg_code[seg];
                    SPAMM_ASSERT(len > 0 && start >= 0 && start + len <= g.task_cap);
                    SPAMM_ASSERT((int64_t)code < (int64_t)g.nb * g.nb);
                }
                mbar_wait(&qempty[q], qphase ^ 1);
                segq[q] = make_int4(seg, len, code, 0);
                mbar_arrive(&qfull[q]);
            }
            seg = __shfl_sync(0xffffffffu, seg, 0);
            start = __shfl_sync(0xffffffffu, start, 0);
            len = __shfl_sync(0xffffffffu, len, 0);
            if (++q == QN) {
                q = 0;
                qphase ^= 1;
            }
            if (seg < 0) break;
            for (int t0 = 0; t0 < len; t0 += 32) {
                const int t = t0 + lane;
                const int sa = t < len ? g.tA[start + t] : 0;
                const int sb = t < len ? g.tB[start + t] : 0;
                const int cnt = len - t0 < 32 ? len - t0 : 32;
                for (int j = 0; j < cnt; j++) {
                    const int a = __shfl_sync(0xffffffffu, sa, j);
                    const int b = __shfl_sync(0xffffffffu, sb, j);
                    SPAMM_ASSERT(a >= 0 && a < g.a_cap);
                    SPAMM_ASSERT(b >= 0 ? b < g.b_cap : (g.peer_world > 0 || (-b - 1) < g.halo_cap));
                    if (lane == 0) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_expect_tx(&full[stage], 2 * TILE_BYTES);
                        bulk_g2s(smem + (2 * stage) * TILE, g.a_pool + (int64_t)a * TILE, TILE_BYTES, &full[stage]);
                        const double *bsrc;
                        if (b >= 0) {
                            bsrc = g.b_pool + (int64_t)b * TILE;
                        } else if (g.peer_world > 0) {   // the owner's pool (peer memory)
                            const int e = -b - 1;
                            bsrc = g.peer_pool[e % g.peer_world] + (int64_t)(e / g.peer_world) * TILE;
                        } else {
                            bsrc = g.b_halo + (int64_t)(-b - 1) * TILE;
                        }
                        bulk_g2s(smem + (2 * stage + 1) * TILE, bsrc, TILE_BYTES, &full[stage]);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        return;
    }

    if (warp > CW) {
        // ------------------------------------------------------- epilogue
        // EW warps copy the deposited tile to the pool (16-byte chunks lane + 32 (ew + EW i):
        // contiguous 512-byte stores per warp instruction); warp 0 of them also sums the
        // consumers' ||C_ij||^2 partials (lane l: lane l of every consumer warp in warp order,
        // then a fixed xor tree; tr over the warps) and writes the block's metadata.
        const int ew = warp - CW - 1;
        uint32_t eph = 0;
        const double2 *eb2 = reinterpret_cast<const double2 *>(ebuf);
        for (;;) {
            mbar_wait(efull, eph);
            eph ^= 1;
            const int4 rec = *erec;
            if (rec.x < 0) break;
            const int seg = rec.x;
            const uint32_t code = (uint32_t)rec.y;
            SPAMM_ASSERT(seg >= 0 && seg < g.c_cap);
            double2 *dst = reinterpret_cast<double2 *>(g.c_pool + (int64_t)seg * TILE);
            constexpr int NCH = TILE / 2 / 32 / EW;   // chunks per lane
            constexpr int NU = NCH < 8 ? NCH : 8;     // loads in flight
#pragma unroll 1
            for (int i0 = 0; i0 < NCH; i0 += NU) {
                double2 v[NU];
#pragma unroll
                for (int j = 0; j < NU; j++) v[j] = eb2[lane + 32 * (ew + EW * (i0 + j))];
#pragma unroll
                for (int j = 0; j < NU; j++) {
                    const int ch = lane + 32 * (ew + EW * (i0 + j)), r = ch / (B / 2), q = ch % (B / 2);
                    dst[r * (B / 2) + (q ^ eswz(r) ^ swz(r))] = v[j];   // to the pool layout
                }
            }
            double ss = 0.0, tr = 0.0;
            const int I = morton_i(code), J = morton_j(code);
            if (ew == 0) {
#pragma unroll
                for (int w = 0; w < CW; w++) ss += ess[32 * w + lane];
                if (!STORE && I == J)
                    for (int w = 0; w < CW; w++) tr += etr[w];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(eempty);   // this warp's reads of the tile are done
            if (ew == 0) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
                if (lane == 0) {
                    g.c_leaf_n2[code] = ss;
                    g.c_coord[seg] = (int32_t)code;
                    g.c_slot[code] = seg;
                    if (!STORE && I == J) g.trace_part[I] = tr;
                }
            }
        }
        return;
    }

    // ----------------------------------------------------------- consumers
    const int g8 = lane >> 2, t4 = lane & 3;
    const int m0 = (warp / WN) * TM, n0 = (warp % WN) * TN;
    // per-thread fragment offsets (doubles) inside a tile; see pool_at / swz
    int aoff[MF][TA ? 4 : 2];
#pragma unroll
    for (int mf = 0; mf < MF; mf++) {
        if constexpr (TA) {
            const int col = m0 + 8 * mf + g8;   // A^T row = A column
#pragma unroll
            for (int s = 0; s < 4; s++)
                aoff[mf][s] = (4 * t4 + s) * B + ((((col >> 1) ^ ((t4 << 1) | (s & 1)))) << 1) + (col & 1);
        } else {
            const int r = m0 + 8 * mf + g8;
#pragma unroll
            for (int h = 0; h < 2; h++) aoff[mf][h] = r * B + (((2 * t4 + h) ^ swz(r)) << 1);
        }
    }
    int boff[NF][4];
#pragma unroll
    for (int nf = 0; nf < NF; nf++) {
        const int col = n0 + 8 * nf + g8;
#pragma unroll
        for (int s = 0; s < 4; s++) boff[nf][s] = (4 * t4 + s) * B + ((((col >> 1) ^ ((t4 << 1) | (s & 1)))) << 1) + (col & 1);
    }

    int stage = 0, q = 0;
    uint32_t phase = 0, qphase = 0, ephase = 0;
    CLK(unsigned long long c_full = 0, c_q = 0, c_bnd = 0, n_task = 0, n_seg = 0, c_map = 0, c_ew = 0;
        const unsigned long long c_start = clock64();)
    for (;;) {
        CLK(unsigned long long c0 = clock64();)
        mbar_wait(&qfull[q], qphase);
        CLK(c_q += clock64() - c0;)
        const int4 e = segq[q];
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[q]);
        if (++q == QN) {
            q = 0;
            qphase ^= 1;
        }
        const int seg = e.x;
        if (seg < 0) break;
        const int len = e.y;
        double acc[MF][NF][2];
#pragma unroll
        for (int i = 0; i < MF; i++)
#pragma unroll
            for (int j = 0; j < NF; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (int it = 0; it < len; it++) {
            // one task: wait for its stage, 16-wide k chunks of fragment loads + DMMAs
            CLK(unsigned long long c1 = clock64();)
            mbar_wait(&full[stage], phase);
            CLK(c_full += clock64() - c1; n_task++;)
            const double *As = smem + (2 * stage) * TILE;
            const double *Bs = As + TILE;
#pragma unroll
            for (int kc = 0; kc < B / 16; kc++) {
                // contraction index permuted inside the 16-wide chunk: k = 16kc + 4t + s
                double a[MF][4], bf[NF][4];
#pragma unroll
                for (int mf = 0; mf < MF; mf++) {
                    if constexpr (TA) {
#pragma unroll
                        for (int s = 0; s < 4; s++) a[mf][s] = As[aoff[mf][s] + 16 * kc * B];
                    } else {
                        const double2 v0 = *reinterpret_cast<const double2 *>(As + aoff[mf][0] + 16 * kc);
                        const double2 v1 = *reinterpret_cast<const double2 *>(As + aoff[mf][1] + 16 * kc);
                        a[mf][0] = v0.x; a[mf][1] = v0.y; a[mf][2] = v1.x; a[mf][3] = v1.y;
                    }
                }
#pragma unroll
                for (int nf = 0; nf < NF; nf++)
#pragma unroll
                    for (int s = 0; s < 4; s++) bf[nf][s] = Bs[boff[nf][s] + 16 * kc * B];
                if (kc == B / 16 - 1) {
                    // Every read of this stage is issued: release it before the last chunk's
                    // DMMAs (which only need registers), so the refill starts a quarter task
                    // earlier and the fence's wait overlaps the previous chunk's DMMAs.  The
                    // refill is a TMA (async-proxy) write: order this thread's generic-proxy
                    // reads before it (cross-proxy WAR).
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[stage]);
                }
#pragma unroll
                for (int s = 0; s < 4; s++)
#pragma unroll
                    for (int mf = 0; mf < MF; mf++)
#pragma unroll
                        for (int nf = 0; nf < NF; nf++)
                            dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], a[mf][s], bf[nf][s]);
            }
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        // the value map and this thread's share of ||C_ij||^2 (and tr X_ii), then deposit
        // the values (eswz layout) and the partials once the epilogue warp has stored the
        // previous tile, and go on to the next segment
        CLK(unsigned long long c4 = clock64(); n_seg++;)
        const uint32_t code = (uint32_t)e.z;
        const bool diag = morton_i(code) == morton_j(code);
        double ssp[MF], trp = 0.0;   // one short FMA chain per mf (the FP64 pipe is busy with DMMAs)
#pragma unroll
        for (int mf = 0; mf < MF; mf++) ssp[mf] = 0.0;
#pragma unroll
        for (int mf = 0; mf < MF; mf++)
#pragma unroll
            for (int nf = 0; nf < NF; nf++) {
                const int r = m0 + 8 * mf + g8, c = n0 + 8 * nf + 2 * t4;
                double y0 = acc[mf][nf][0], y1 = acc[mf][nf][1];
                if (EPI == EPI_STORE_SCALED) {   // the fused final unscale of an NS run
                    y0 *= g.alpha;
                    y1 *= g.alpha;
                }
                if (!STORE && diag) {
                    if (r == c) trp += y0;
                    if (r == c + 1) trp += y1;
                }
                if (EPI == EPI_NS_H) {
                    // H = 1/2 (3 delta - X) written as 1.5 delta - 0.5 x (the 1/2 is exact)
                    const double d0 = (diag && r == c) ? 1.5 : 0.0, d1 = (diag && r == c + 1) ? 1.5 : 0.0;
                    y0 = d0 - 0.5 * y0;
                    y1 = d1 - 0.5 * y1;
                }
                ssp[mf] = fma(y0, y0, ssp[mf]);
                ssp[mf] = fma(y1, y1, ssp[mf]);
                acc[mf][nf][0] = y0;
                acc[mf][nf][1] = y1;
            }
        if (!STORE && diag) {   // warp-uniform, ~1 segment in 100 at C5
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) trp += __shfl_xor_sync(0xffffffffu, trp, o);
        }
        CLK(unsigned long long c5 = clock64();)
        mbar_wait(eempty, ephase ^ 1);
        CLK(unsigned long long c6 = clock64(); c_map += c5 - c4; c_ew += c6 - c5;)
        ephase ^= 1;
#pragma unroll
        for (int mf = 0; mf < MF; mf++)
#pragma unroll
            for (int nf = 0; nf < NF; nf++) {
                const int r = m0 + 8 * mf + g8, c = n0 + 8 * nf + 2 * t4;
                reinterpret_cast<double2 *>(ebuf)[r * (B / 2) + ((c >> 1) ^ eswz(r))] =
                    make_double2(acc[mf][nf][0], acc[mf][nf][1]);
            }
#pragma unroll
        for (int w = MF / 2; w > 0; w >>= 1)   // fixed pairwise tree
#pragma unroll
            for (int mf = 0; mf < w; mf++) ssp[mf] += ssp[mf + w];
        ess[32 * warp + lane] = ssp[0];
        if (!STORE && diag && lane == 0) etr[warp] = trp;
        __syncwarp();
        if (lane == 0) {
            if (warp == 0) *erec = make_int4(seg, e.z, 0, 0);
            mbar_arrive(efull);
        }
        CLK(c_bnd += clock64() - c4;)
    }
    // end of the launch: tell the epilogue warp (after its last tile is read)
    mbar_wait(eempty, ephase ^ 1);
    __syncwarp();
    if (lane == 0) {
        if (warp == 0) *erec = make_int4(-1, 0, 0, 0);
        mbar_arrive(efull);
    }
    CLK(if (lane == 0) {
        atomicAdd(&g_gemm_clk[0], clock64() - c_start);
        atomicAdd(&g_gemm_clk[1], c_full);
        atomicAdd(&g_gemm_clk[2], c_q);
        atomicAdd(&g_gemm_clk[3], c_bnd);
        atomicAdd(&g_gemm_clk[4], n_task);
        atomicAdd(&g_gemm_clk[5], n_seg);
        atomicAdd(&g_gemm_clk[6], c_map);
        atomicAdd(&g_gemm_clk[7], c_ew);
    })
}

template <int B, int CW, int WM, int WN, int STAGES, int EPI, int TA>
static spamm_status launch_gemm(spamm_ctx ctx, const GemmArgs &g)
{
    constexpr int NT = 32 * (CW + 1 + EW);
    const size_t smem = GemmSmem<B, CW, STAGES>::bytes;
    auto kern = k_leaf_gemm<B, CW, WM, WN, STAGES, EPI, TA>;
    static std::atomic<uint64_t> configured{0};
    static std::atomic<int> occ_cache{0};
    CK(once_per_device(configured, ctx->device, [&]() {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int o = 0;
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, NT, smem);
        if (e == cudaSuccess) occ_cache.store(o < 1 ? 1 : o);
        return e;
    }));
    if (g.nseg == 0 && !g.nseg_dev) return SPAMM_OK;
    const int occ = occ_cache.load();
    int grid = ctx->sm_count * occ;
    if (!g.nseg_dev && grid > g.nseg) grid = g.nseg;
    if (ctx->gemm_grid_cap > 0 && grid > ctx->gemm_grid_cap) grid = ctx->gemm_grid_cap;
    kern<<<grid, NT, smem, ctx->stream>>>(g);
    CKL(ctx);
    return SPAMM_OK;
}

template <int EPI, int TA>
static spamm_status gemm_dispatch(spamm_ctx ctx, int b, const GemmArgs &g)
{
    switch (b) {
    case 64: return launch_gemm<64, 8, 2, 4, 3, EPI, TA>(ctx, g);
    case 32: return launch_gemm<32, 4, 2, 2, 4, EPI, TA>(ctx, g);
    case 16: return launch_gemm<16, 1, 1, 1, 4, EPI, TA>(ctx, g);
    default: return set_err(ctx, SPAMM_EINVAL, "b=%d", b);
    }
}

spamm_status gemm_run(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, const double *b_halo,
                      spamm_mat C, int epi, double *trace_part, const int32_t *seg_order, int64_t nseg,
                      int ticket, int transA, bool device_count)
{
    if (nseg < 0) nseg = cw->nsegs;
    GemmArgs g{A->pool, B->pool, b_halo, cw->tA, cw->tB, cw->seg_code, cw->seg_start, cw->seg_len,
               (int)nseg, seg_order, C->pool, C->coord, C->slot, C->norm2 + pyr_off(C->L), trace_part,
               cw->counters + CNT_GEMM_TICKET + ticket, cw->alpha,
               device_count ? cw->counters + CNT_NSEG : nullptr, cw->peer_world, {},
               A->cap, B->cap, b_halo ? (int64_t)1 << 40 : 0, C->cap, cw->cap, cw->cap_segs, A->nb};
    for (int q = 0; q < cw->peer_world; q++) g.peer_pool[q] = cw->peer_pool[q];
    if (transA) {
        if (epi == EPI_NS_H) return gemm_dispatch<EPI_NS_H, 1>(ctx, A->b, g);
        if (epi == EPI_NS_X) return gemm_dispatch<EPI_NS_X, 1>(ctx, A->b, g);
        if (g.alpha != 1.0) return gemm_dispatch<EPI_STORE_SCALED, 1>(ctx, A->b, g);
        return gemm_dispatch<EPI_STORE, 1>(ctx, A->b, g);
    }
    if (epi == EPI_NS_H) return gemm_dispatch<EPI_NS_H, 0>(ctx, A->b, g);
    if (epi == EPI_NS_X) return gemm_dispatch<EPI_NS_X, 0>(ctx, A->b, g);
    if (g.alpha != 1.0) return gemm_dispatch<EPI_STORE_SCALED, 0>(ctx, A->b, g);
    return gemm_dispatch<EPI_STORE, 0>(ctx, A->b, g);
}

// ------------------------------------------------------- LPT segment order
// The persistent GEMM takes segments from a ticket; running the longest first
// bounds the tail of a launch by the shortest segments (longest-processing-time
// first).  The order is only a schedule: every segment is owned by one CTA and
// accumulated in ascending k whatever its position, so results do not depend on
// it (positions inside a length bucket are taken with atomics).
constexpr int LPT_BUCKETS = 1024;

__global__ void k_lpt_hist(const int32_t *in, int64_t n, const int32_t *seg_len, int32_t *hist)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int s = in ? in[q] : (int)q;
    const int len = seg_len[s];
    atomicAdd(&hist[len < LPT_BUCKETS ? len : LPT_BUCKETS - 1], 1);
}

// single CTA: base[len] = number of segments longer than len (descending order)
__global__ void __launch_bounds__(LPT_BUCKETS) k_lpt_scan(int32_t *hist)
{
    __shared__ V1 sw[LPT_BUCKETS / 32];
    const int t = threadIdx.x;                 // t-th bucket from the top
    const int bkt = LPT_BUCKETS - 1 - t;
    V1 v{hist[bkt]};
    V1 tot;
    V1 ex = block_excl_scan<V1, LPT_BUCKETS>(v, &tot, sw);
    hist[bkt] = ex.x;
}

__global__ void k_lpt_scatter(const int32_t *in, int64_t n, const int32_t *seg_len, int32_t *base, int32_t *out)
{
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int s = in ? in[q] : (int)q;
    const int len = seg_len[s];
    out[atomicAdd(&base[len < LPT_BUCKETS ? len : LPT_BUCKETS - 1], 1)] = s;
}

spamm_status lpt_order(spamm_ctx ctx, const int32_t *seg_len, const int32_t *in, int64_t n, int32_t *out)
{
    if (n <= 0) return SPAMM_OK;
    int32_t *hist = dalloc<int32_t>(ctx, LPT_BUCKETS);
    if (!hist) return set_err(ctx, SPAMM_ENOMEM, "lpt histogram");
    CK(cudaMemsetAsync(hist, 0, sizeof(int32_t) * LPT_BUCKETS, ctx->stream));
    k_lpt_hist<<<cdiv(n, 256), 256, 0, ctx->stream>>>(in, n, seg_len, hist);
    CKL(ctx);
    k_lpt_scan<<<1, LPT_BUCKETS, 0, ctx->stream>>>(hist);
    CKL(ctx);
    k_lpt_scatter<<<cdiv(n, 256), 256, 0, ctx->stream>>>(in, n, seg_len, hist, out);
    CKL(ctx);
    dev_free(ctx, hist, sizeof(int32_t) * LPT_BUCKETS);
    return SPAMM_OK;
}

// -------------------------------------------------- diagonal fix-up of H
// H_ii = 1.5 I where X had no surviving task (i,i) (K6): slots appended at
// nseg.. in ascending i (single-CTA scan, deterministic), then filled in parallel.
template <int THREADS>
__global__ void k_diag_assign(int32_t *slot_map, int32_t *coord, int nb, int r0, int r1, int64_t base,
                              int32_t *newslot, int64_t *count_out, const int32_t *base_dev, int64_t cap)
{
    pdl_wait();
    pdl_trigger();
    __shared__ V1 sw[THREADS / 32];
    if (base_dev) base = *base_dev;   // device-driven step: after the X product's segments
    int64_t run = 0;
    for (int i0 = 0; i0 < nb; i0 += THREADS) {
        int i = i0 + threadIdx.x;
        uint32_t code = i < nb ? morton(i, i) : 0;
        V1 v{(i >= r0 && i < r1 && slot_map[code] < 0) ? 1 : 0};
        V1 tot;
        V1 ex = block_excl_scan<V1, THREADS>(v, &tot, sw);
        if (i < nb) {
            int32_t s = v.x ? (int32_t)(base + run + ex.x) : -1;
            SPAMM_ASSERT(s < 0 || s < cap);
            newslot[i] = s;
            if (v.x) {
                slot_map[code] = s;
                coord[s] = (int32_t)code;
            }
        }
        run += tot.x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *count_out = run;
}

// trace_part != nullptr: CTA 0 also forms t = (n - sum_i trace_part[i]) / n exactly as
// k_trace_finish does (256 threads, i strided by 256, then the halving tree) -- one launch
// fewer per NS step (the trace partials are complete once the X GEMM is)
__device__ __forceinline__ void trace_256(const double *part, int nb, double n, double *t_out)
{
    __shared__ double sh[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += 256) s += part[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *t_out = (n - sh[0]) / n;
}

__global__ void __launch_bounds__(256) k_diag_fill(const int32_t *newslot, double *pool, int b, double value,
                                                   double *leaf_n2, const double *trace_part, int nb, double n,
                                                   double *t_out)
{
    pdl_wait();
    pdl_trigger();
    int i = blockIdx.x;
    if (trace_part && i == 0) trace_256(trace_part, nb, n, t_out);
    int s = newslot[i];
    if (s < 0) return;
    double *d = pool + (int64_t)s * b * b;
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) d[e] = (e / b == pool_col(e, b)) ? value : 0.0;
    if (threadIdx.x == 0) {
        double ss = 0.0;
        for (int r = 0; r < b; r++) ss += value * value;
        leaf_n2[morton(i, i)] = ss;
    }
}

spamm_status diag_append(spamm_ctx ctx, spamm_mat m, int64_t base, double value, int64_t *added)
{
    int32_t *newslot = dalloc<int32_t>(ctx, m->nb);
    if (!newslot) return set_err(ctx, SPAMM_ENOMEM, "diag fixup");
    CK(launch_k(ctx, k_diag_assign<1024>, 1, 1024, 0, m->slot, m->coord, m->nb, m->r0, m->r1, base, newslot,
                ctx->iscratch, (const int32_t *)nullptr, m->cap));
    CKL(ctx);
    CK(launch_k(ctx, k_diag_fill, m->nb, 256, 0, (const int32_t *)newslot, m->pool, m->b, value,
                m->norm2 + pyr_off(m->L), (const double *)nullptr, 0, 0.0, (double *)nullptr));
    CKL(ctx);
    int64_t h = 0;
    ST(fetch1(ctx, ctx->iscratch, &h, sizeof(int64_t)));
    dev_free(ctx, newslot, sizeof(int32_t) * m->nb);
    *added = h;
    return SPAMM_OK;
}

spamm_status diag_fixup_async(spamm_ctx ctx, spamm_mat H, int64_t nseg, double value, int64_t *dcount,
                              const double *trace_part, double *t_out)
{
    int32_t *newslot = dalloc<int32_t>(ctx, H->nb);
    if (!newslot) return set_err(ctx, SPAMM_ENOMEM, "diag fixup");
    CK(launch_k(ctx, k_diag_assign<1024>, 1, 1024, 0, H->slot, H->coord, H->nb, H->r0, H->r1, nseg, newslot, dcount,
                (const int32_t *)nullptr, H->cap));
    CKL(ctx);
    CK(launch_k(ctx, k_diag_fill, H->nb, 256, 0, (const int32_t *)newslot, H->pool, H->b, value,
                H->norm2 + pyr_off(H->L), trace_part, H->nb, (double)H->n, t_out));
    CKL(ctx);
    dev_free(ctx, newslot, sizeof(int32_t) * H->nb);
    H->nblk = nseg;   // provisional until the caller has fetched *dcount
    return SPAMM_OK;
}

spamm_status diag_fixup_dev(spamm_ctx ctx, spamm_mat H, const int32_t *nseg_dev, double value, int32_t *newslot,
                            int64_t *dcount, const double *trace_part, double *t_out)
{
    CK(launch_k(ctx, k_diag_assign<1024>, 1, 1024, 0, H->slot, H->coord, H->nb, H->r0, H->r1, (int64_t)0, newslot,
                dcount, nseg_dev, H->cap));
    CKL(ctx);
    CK(launch_k(ctx, k_diag_fill, H->nb, 256, 0, (const int32_t *)newslot, H->pool, H->b, value,
                H->norm2 + pyr_off(H->L), trace_part, H->nb, (double)H->n, t_out));
    CKL(ctx);
    return SPAMM_OK;
}

spamm_status diag_fixup(spamm_ctx ctx, spamm_mat H, int64_t nseg, double value)
{
    int64_t added = 0;
    ST(diag_append(ctx, H, nseg, value, &added));
    H->nblk = nseg + added;
    return SPAMM_OK;
}

// t = (n - sum_i trace_part[i]) / n, fixed-order single-CTA reduction
__global__ void __launch_bounds__(256) k_trace_finish(const double *part, int nb, double n, double *t_out)
{
    pdl_wait();
    pdl_trigger();
    trace_256(part, nb, n, t_out);
}

spamm_status trace_finish(spamm_ctx ctx, const double *trace_part, int nb, int64_t n, double *t_out)
{
    CK(launch_k(ctx, k_trace_finish, 1, 256, 0, trace_part, nb, (double)n, t_out));
    CKL(ctx);
    return SPAMM_OK;
}

// ------------------------------------------- scaled / stabilised NS map
// alpha(t) = 1 + 1.85 (1 + e^{-50(t-.35)})^{-1}, eps(t) = .1 (1 + e^{-75(t-.30)})^{-1},
// computed on the device from t_k (no host round trip).  coef = {alpha, eps, sqrt(alpha)/2}.
__global__ void k_ns_coef(const double *t, double *coef)
{
    const double tk = *t;
    const double a = 1.0 + 1.85 * (1.0 / (1.0 + exp(-50.0 * (tk - 0.35))));
    const double e = 0.1 * (1.0 / (1.0 + exp(-75.0 * (tk - 0.30))));
    coef[0] = a;
    coef[1] = e;
    coef[2] = sqrt(a) / 2.0;
}

// In place over the stored X blocks: x~ = (1 - 2 eps) x + eps delta ("[0,1] -> [eps, 1-eps]
// prior to the logistic"), H = sqrt(alpha)/2 (3 delta - alpha x~); ||H_ij||^2 to the leaf
// level (thread partials in element order, then a fixed tree: deterministic).
__global__ void __launch_bounds__(256) k_ns_map(double *pool, const int32_t *coord, int b, const double *coef,
                                                double *leaf_n2)
{
    __shared__ double red[256];
    const int64_t blk = blockIdx.x;
    const uint32_t code = coord[blk];
    const bool diag = morton_i(code) == morton_j(code);
    const double a = coef[0], e = coef[1], sa = coef[2];
    double *p = pool + blk * (int64_t)b * b;
    double ss = 0.0;
    for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
        const int r = idx / b, q = pool_col(idx, b);
        const double d = (diag && r == q) ? 1.0 : 0.0;
        const double xt = (1.0 - 2.0 * e) * p[idx] + e * d;
        const double h = sa * (3.0 * d - a * xt);
        p[idx] = h;
        ss = fma(h, h, ss);
    }
    red[threadIdx.x] = ss;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) leaf_n2[code] = red[0];
}

spamm_status ns_scaled_map(spamm_ctx ctx, spamm_mat X, const double *t, double *coef)
{
    k_ns_coef<<<1, 1, 0, ctx->stream>>>(t, coef);
    CKL(ctx);
    if (X->nblk > 0) {
        k_ns_map<<<(int)X->nblk, 256, 0, ctx->stream>>>(X->pool, X->coord, X->b, coef, X->norm2 + pyr_off(X->L));
        CKL(ctx);
    }
    return SPAMM_OK;
}
