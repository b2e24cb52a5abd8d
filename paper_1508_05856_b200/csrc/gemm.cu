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
//     of ||C_ij||^2 (and tr X_ii) in short FMA chains, hand the values and the partial
//     to the epilogue warps and go on to the next segment.
//   warps CW+1 .. CW+EW (epilogue): store the handed-off tile to the pool; the first
//     also sums the consumers' partials in a fixed order (deterministic) and writes
//     the block's metadata.
// The consumers issue no global stores, shuffle trees or cross-warp hand-offs, so
// the DMMA pipe keeps running across segment boundaries.  The hand-off (EpiCfg):
//   b = 64: through tensor memory, NBUF = 4 tiles deep — one tcgen05.st (STTM.x32) per
//     consumer thread, one epilogue warp per SM sub-partition reading its lanes back
//     (LDTM.x32) and storing whole 128-byte lines.  Measured on the C5 / C3 k = 8 NS
//     steps (tools/gemm_probe.py): GEMM 59.37 / 5.496 ms against 59.56 / 5.511 ms with
//     the single shared-memory tile (its wait for the previous tile's store, 0.7 % of
//     the consumers' cycles, is gone); the epilogue warps poll with a 512 ns sleep
//     (spinning: 60.26 ms, they share the producer's sub-partition) and must store
//     whole lines (8 rows x 64 bytes per instruction: 59.86 ms).
//   b = 32 / 16: one shared-memory tile (eswz layout), EW = 2 epilogue warps copying
//     it with contiguous 16-byte stores.  For b = 64 this was the round-2 design before
//     TMEM: EW = 2 measured best (EW = 1: +0.1 %, EW = 4: +0.7 %); a single epilogue
//     warp that also did the map and norms fell behind (the FP64 pipe is busy with
//     DMMAs), and a TMA bulk store of the tile needs a proxy fence in every consumer
//     thread (5.6 % of their cycles at the boundary).
// TA = 1: the left operand is A^T (single channel, §8(f) f2): the A tile is read
// with the column pattern of the B fragments (A^T[m][k] = A[k][m]).
// The epilogue tile's own chunk swizzle: chunk c/2 of row r at (c/2) ^ eswz(r).  A deposit
// instruction (rows 8mf + g8, chunks 4nf + t4 + const) then fills 8 distinct 16-byte bank
// slots in each 8-lane phase (the pool swizzle would put rows 2p and 2p+1 on the same 4:
// two-way conflicts); the epilogue warps read whole rows and store them in the pool layout.
__device__ __forceinline__ int eswz(int r) { return (r & 1) << 2; }

#ifndef SPAMM_EPI_WARPS
#define SPAMM_EPI_WARPS 2
#endif
#ifndef SPAMM_EPI_TMEM
#define SPAMM_EPI_TMEM 1
#endif
#ifndef SPAMM_SMEM_NBUF
#define SPAMM_SMEM_NBUF 1   // shared-memory epilogue tiles (b = 32 / 16)
#endif
#ifndef SPAMM_B32_STAGES
#define SPAMM_B32_STAGES 4
#endif
#ifndef SPAMM_EPI_SLEEP
#define SPAMM_EPI_SLEEP 512   // ns between the epilogue warps' probes of the next tile; 0 = spin
#endif
// Epilogue hand-off.  b = 64 (8 consumer warps, 32x16 warp tiles): the finished tile goes
// through tensor memory — each consumer warp writes its 16 values per thread with one
// tcgen05.st into the TMEM lanes of its SM sub-partition, and one epilogue warp per
// sub-partition (warp id mod 4 selects the lanes a warp may access) reads them back with
// tcgen05.ld and stores them to the pool.  TMEM (256 KB per SM, otherwise unused here: FP64
// has no tcgen05.mma kind) holds NBUF tiles, so a consumer never waits for the previous tile
// to be stored.  Other b: one shared-memory tile, EW epilogue warps.
template <int B, int CW>
struct EpiCfg {
    static constexpr bool TE = SPAMM_EPI_TMEM && B == 64 && CW == 8;
    static constexpr int EW = TE ? 4 : SPAMM_EPI_WARPS;   // epilogue warps
    static constexpr int NBUF = TE ? 4 : SPAMM_SMEM_NBUF;  // tiles in flight to the epilogue warps
    static constexpr uint32_t TCOLS = TE ? 64 * NBUF : 0;  // TMEM columns (b32) allocated
};

template <int B, int CW, int STAGES>
struct GemmSmem {
    static constexpr int TILE = B * B;
    static constexpr int QN = 4;   // segment-queue depth (producer -> consumers)
    static constexpr int NBUF = EpiCfg<B, CW>::NBUF;
    // doubles: STAGES x {A, B} tiles, the epilogue tile (not with TMEM), per buffer the
    // consumers' per-lane ||.||^2 partials and per-warp trace partials; then the barriers,
    // the queue, the records and the TMEM base address
    static constexpr int ETR = (CW + 1) & ~1;   // tr partials, padded to keep 16-byte alignment
    static constexpr size_t bytes =
        sizeof(double) * ((2 * STAGES + (EpiCfg<B, CW>::TE ? 0 : NBUF)) * TILE + NBUF * (32 * CW + ETR)) +
        sizeof(uint64_t) * (2 * STAGES + 2 * QN + 2 * NBUF) + sizeof(int4) * (QN + NBUF + 1);
    static_assert(bytes <= 227 * 1024, "the leaf GEMM's shared memory exceeds the 227 KiB an sm_100a CTA may use");
};

// ---- tensor memory (tcgen05) helpers for the TMEM epilogue hand-off
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
#define TM_R32(p)                                                                                          \
    "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]), "r"(p[6]), "r"(p[7]), "r"(p[8]),     \
        "r"(p[9]), "r"(p[10]), "r"(p[11]), "r"(p[12]), "r"(p[13]), "r"(p[14]), "r"(p[15]), "r"(p[16]),      \
        "r"(p[17]), "r"(p[18]), "r"(p[19]), "r"(p[20]), "r"(p[21]), "r"(p[22]), "r"(p[23]), "r"(p[24]),     \
        "r"(p[25]), "r"(p[26]), "r"(p[27]), "r"(p[28]), "r"(p[29]), "r"(p[30]), "r"(p[31])
#define TM_W32(p)                                                                                          \
    "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]), "=r"(p[7]),        \
        "=r"(p[8]), "=r"(p[9]), "=r"(p[10]), "=r"(p[11]), "=r"(p[12]), "=r"(p[13]), "=r"(p[14]),           \
        "=r"(p[15]), "=r"(p[16]), "=r"(p[17]), "=r"(p[18]), "=r"(p[19]), "=r"(p[20]), "=r"(p[21]),         \
        "=r"(p[22]), "=r"(p[23]), "=r"(p[24]), "=r"(p[25]), "=r"(p[26]), "=r"(p[27]), "=r"(p[28]),         \
        "=r"(p[29]), "=r"(p[30]), "=r"(p[31])
#define TM_ARGS32                                                                                          \
    "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28," \
    "%29,%30,%31,%32}"
// thread l of the warp: 32 consecutive b32 columns of TMEM lane (taddr.lane + l)
__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t (&v)[32])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], " TM_ARGS32 ";\n" ::"r"(taddr), TM_R32(v)
                 : "memory");
}
__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&v)[32])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,"
                 "%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                 : TM_W32(v)
                 : "r"(taddr)
                 : "memory");
}

// GRP = 1: two products in one launch (the Y' and Z' products of a captured NS step, both plain
// stores): tickets [0, n1) are g's segments, [n1, n1 + n2) g2's; the segment's product rides in
// the queue entry and the epilogue record.  Single device only (no halo / peer tiles).
template <int B, int CW, int WM, int WN, int STAGES, int EPI, int TA, int GRP = 0>
__global__ void __launch_bounds__(32 * (CW + 1 + EpiCfg<B, CW>::EW), 1) k_leaf_gemm(GemmArgs g, GemmArgs g2)
{
    static_assert(!GRP || (EPI == EPI_STORE && TA == 0), "grouped launches: plain-store products");
    static_assert(WM * WN == CW, "warp grid");
    constexpr bool STORE = EPI == EPI_STORE || EPI == EPI_STORE_SCALED;
    constexpr int TM = B / WM, TN = B / WN;
    constexpr int MF = TM / 8, NF = TN / 8;
    constexpr int TILE = B * B;
    constexpr uint32_t TILE_BYTES = TILE * 8;
    constexpr bool TE = EpiCfg<B, CW>::TE;
    constexpr int EW = EpiCfg<B, CW>::EW, NBUF = EpiCfg<B, CW>::NBUF;
    // TMEM hand-off: consumer warp w writes lanes 32 (w mod 4).. of columns 64 buf + 32 (w / 4)..;
    // that needs the two consumer warps of a sub-partition to be warps w, w + 4 (WN = 4) and
    // 16 values = 32 b32 columns per thread
    static_assert(!TE || (WN == 4 && CW == 8 && MF * NF * 4 == 32 && EW == 4), "TMEM epilogue layout");
    extern __shared__ __align__(1024) double smem[];
    constexpr int QN = GemmSmem<B, CW, STAGES>::QN;
    constexpr int ETR = GemmSmem<B, CW, STAGES>::ETR;
    double *ebuf = smem + 2 * STAGES * TILE;                  // [NBUF] epilogue tiles (eswz layout; not with TMEM)
    double *ess = ebuf + (TE ? 0 : NBUF * TILE);              // [NBUF][CW][32] lanes' ||C_ij||^2 partials
    double *etr = ess + NBUF * 32 * CW;                       // [NBUF][ETR] warps' tr partials (diagonal blocks)
    uint64_t *full = reinterpret_cast<uint64_t *>(etr + NBUF * ETR);
    uint64_t *empty = full + STAGES;
    uint64_t *qfull = empty + STAGES;
    uint64_t *qempty = qfull + QN;
    uint64_t *efull = qempty + QN;                            // [NBUF] tile deposited (CW arrivals)
    uint64_t *eempty = efull + NBUF;                          // [NBUF] tile stored by the epilogue warps
    int4 *segq = reinterpret_cast<int4 *>(eempty + NBUF);     // {seg, len, code, -} per queue entry
    int4 *erec = segq + QN;                                   // [NBUF] {seg, code} of the deposited tile
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(erec + NBUF);

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
        for (int e = 0; e < NBUF; e++) {
            mbar_init(&efull[e], CW);
            mbar_init(&eempty[e], EW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if constexpr (TE) {
        // the first epilogue warp owns the allocation (and frees it at the end); one CTA per SM
        // (the stage ring alone takes 192 KiB), so the columns are always free
        if (warp == CW + 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_u32(tmem_slot)),
                         "n"(EpiCfg<B, CW>::TCOLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
        }
        tm_fence_before();
    }
    __syncthreads();
    uint32_t tbase = 0;
    if constexpr (TE) {
        tm_fence_after();
        tbase = *tmem_slot;
    }

    if (warp == CW) {
        // ------------------------------------------------------- producer
        // Dynamic scheduling: segments (Morton order) are taken from a global
        // ticket and announced to the consumers through a QN-deep smem queue.
        int stage = 0, q = 0;
        uint32_t phase = 0, qphase = 0;
        for (;;) {
            int seg = 0, start = 0, len = 0, pp = 0;
            if (lane == 0) {
                seg = atomicAdd(g.ticket, 1);
                const int lim = g.nseg_dev ? *g.nseg_dev : g.nseg;
                if (seg >= lim) {
                    seg -= lim;
                    pp = 1;
                    if (!GRP || seg >= (g2.nseg_dev ? *g2.nseg_dev : g2.nseg)) seg = -1;
                } else if (g.seg_order) {
                    seg = g.seg_order[seg];
                }
                int code = 0;
                if (seg >= 0) {
                    const GemmArgs &gp = (GRP && pp) ? g2 : g;
                    SPAMM_ASSERT(seg < gp.seg_cap);
                    start = gp.seg_start[seg];
                    len = gp.seg_len[seg];
                    code = gp.seg_code[seg];
                    SPAMM_ASSERT(len > 0 && start >= 0 && start + len <= gp.task_cap);
                    SPAMM_ASSERT((int64_t)code < (int64_t)gp.nb * gp.nb);
                }
                mbar_wait(&qempty[q], qphase ^ 1);
                segq[q] = make_int4(seg, len, code, pp);
                mbar_arrive(&qfull[q]);
            }
            seg = __shfl_sync(0xffffffffu, seg, 0);
            start = __shfl_sync(0xffffffffu, start, 0);
            len = __shfl_sync(0xffffffffu, len, 0);
            if (GRP) pp = __shfl_sync(0xffffffffu, pp, 0);
            const int32_t *tAp = (GRP && pp) ? g2.tA : g.tA, *tBp = (GRP && pp) ? g2.tB : g.tB;
            const double *apool = (GRP && pp) ? g2.a_pool : g.a_pool, *bpool = (GRP && pp) ? g2.b_pool : g.b_pool;
            if (++q == QN) {
                q = 0;
                qphase ^= 1;
            }
            if (seg < 0) break;
            for (int t0 = 0; t0 < len; t0 += 32) {
                const int t = t0 + lane;
                const int sa = t < len ? tAp[start + t] : 0;
                const int sb = t < len ? tBp[start + t] : 0;
                const int cnt = len - t0 < 32 ? len - t0 : 32;
                for (int j = 0; j < cnt; j++) {
                    const int a = __shfl_sync(0xffffffffu, sa, j);
                    const int b = __shfl_sync(0xffffffffu, sb, j);
                    SPAMM_ASSERT(a >= 0 && a < ((GRP && pp) ? g2.a_cap : g.a_cap));
                    SPAMM_ASSERT(b >= 0 ? b < ((GRP && pp) ? g2.b_cap : g.b_cap)
                                        : (!GRP && (g.peer_world > 0 || (-b - 1) < g.halo_cap)));
                    if (lane == 0) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_expect_tx(&full[stage], 2 * TILE_BYTES);
                        bulk_g2s(smem + (2 * stage) * TILE, apool + (int64_t)a * TILE, TILE_BYTES, &full[stage]);
                        const double *bsrc;
                        if (b >= 0) {
                            bsrc = bpool + (int64_t)b * TILE;
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
        // Shared-memory tile: EW warps copy it to the pool (16-byte chunks lane + 32 (ew + EW i):
        // contiguous 512-byte stores per warp instruction).  TMEM: the warp of sub-partition
        // qd = warp mod 4 loads the values consumer warps qd and qd + 4 wrote into its lanes
        // (thread l: lane l's 16 values of each) and stores them in the pool layout (8 rows x
        // 64 contiguous bytes per warp instruction).  Epilogue warp 0 also sums the consumers'
        // ||C_ij||^2 partials (lane l: lane l of every consumer warp in warp order, then a fixed
        // xor tree; tr over the warps) and writes the block's metadata.
        const int ew = warp - CW - 1;
        const int g8 = lane >> 2, t4 = lane & 3;
        uint32_t eph = 0;
        int eb = 0;
        for (;;) {
            // (TMEM ring: 4 tiles deep, the store is off the critical path; the single shared-
            // memory tile of b = 32 / 16 is waited for by the consumers: spin)
            if (TE && SPAMM_EPI_SLEEP > 0) mbar_wait_sleep(&efull[eb], eph, SPAMM_EPI_SLEEP);
            else mbar_wait(&efull[eb], eph);
            if constexpr (TE) tm_fence_after();
            const int4 rec = erec[eb];
            if (rec.x < 0) break;
            const int seg = rec.x;
            const uint32_t code = (uint32_t)rec.y;
            const bool p2 = GRP && rec.z;   // grouped launch: the segment's product
            SPAMM_ASSERT(seg >= 0 && seg < (p2 ? g2.c_cap : g.c_cap));
            double2 *dst = reinterpret_cast<double2 *>((p2 ? g2.c_pool : g.c_pool) + (int64_t)seg * TILE);
            uint32_t tv[TE ? 2 : 1][32];
            if constexpr (TE) {
                const int qd = warp & 3;
                tm_ld32(tbase + ((uint32_t)(32 * qd) << 16) + 64 * eb, tv[0]);
                tm_ld32(tbase + ((uint32_t)(32 * qd) << 16) + 64 * eb + 32, tv[TE ? 1 : 0]);
                tm_wait_ld();
            } else {
                const double2 *eb2 = reinterpret_cast<const double2 *>(ebuf + eb * TILE);
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
            }
            double ss = 0.0, tr = 0.0;
            const int I = morton_i(code), J = morton_j(code);
            if (ew == 0) {
                const double *es = ess + eb * 32 * CW;
#pragma unroll
                for (int w = 0; w < CW; w++) ss += es[32 * w + lane];
                if (!STORE && I == J)
                    for (int w = 0; w < CW; w++) tr += etr[eb * ETR + w];
            }
            if constexpr (TE) tm_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&eempty[eb]);   // this warp's reads of the tile are done
            if constexpr (TE) {
                // This warp's columns [16 qd, 16 qd + 16) are one 128-byte line of each row (the
                // pool swizzle permutes 16-byte chunks inside aligned 128-byte groups).  Lane
                // (g8, t4) holds chunks t4 (nf = 0) and 4 + t4 (nf = 1) of row 8 mf + g8; after one
                // exchange with lane ^ 16 (g8 ^ 4) each store instruction writes 4 whole lines:
                // rows 0..3 of the 8-row group first, then rows 4..7.
                const bool lo = g8 < 4;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int cw = (warp & 3) + 4 * h;   // the consumer warp whose values tv[h] holds
                    const int m0 = (cw / WN) * TM, n0 = (cw % WN) * TN;
#pragma unroll
                    for (int mf = 0; mf < MF; mf++) {
                        const int j0 = 4 * (mf * NF), j1 = 4 * (mf * NF + 1);
                        const double2 v0 = make_double2(__hiloint2double((int)tv[h][j0 + 1], (int)tv[h][j0]),
                                                        __hiloint2double((int)tv[h][j0 + 3], (int)tv[h][j0 + 2]));
                        double2 v1 = make_double2(__hiloint2double((int)tv[h][j1 + 1], (int)tv[h][j1]),
                                                  __hiloint2double((int)tv[h][j1 + 3], (int)tv[h][j1 + 2]));
                        v1.x = __shfl_xor_sync(0xffffffffu, v1.x, 16);   // now the partner's nf = 1 values
                        v1.y = __shfl_xor_sync(0xffffffffu, v1.y, 16);
                        const int rbase = m0 + 8 * mf;
                        // first: rows rbase + 0..3 (own nf = 0 if g8 < 4, else the partner's nf = 1)
                        const int ra = rbase + (g8 & 3), rb = ra + 4;
                        const int ca = n0 + (lo ? 2 * t4 : 8 + 2 * t4), cb = n0 + (lo ? 8 + 2 * t4 : 2 * t4);
                        dst[ra * (B / 2) + ((ca >> 1) ^ swz(ra))] = lo ? v0 : v1;
                        dst[rb * (B / 2) + ((cb >> 1) ^ swz(rb))] = lo ? v1 : v0;
                    }
                }
            }
            if (ew == 0) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
                if (lane == 0) {
                    (p2 ? g2.c_leaf_n2 : g.c_leaf_n2)[code] = ss;
                    (p2 ? g2.c_coord : g.c_coord)[seg] = (int32_t)code;
                    (p2 ? g2.c_slot : g.c_slot)[code] = seg;
                    if (!STORE && I == J) g.trace_part[I] = tr;
                }
            }
            if (++eb == NBUF) {
                eb = 0;
                eph ^= 1;
            }
        }
        if constexpr (TE) {
            // every epilogue warp's last TMEM read is done before the owner frees the columns
            tm_fence_before();
            asm volatile("bar.sync 1, %0;\n" ::"n"(32 * EW) : "memory");
            if (ew == 0) {
                tm_fence_after();
                asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase),
                             "n"(EpiCfg<B, CW>::TCOLS)
                             : "memory");
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
    int eb = 0;   // epilogue buffer
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
        mbar_wait(&eempty[eb], ephase ^ 1);
        CLK(unsigned long long c6 = clock64(); c_map += c5 - c4; c_ew += c6 - c5;)
        if constexpr (TE) {
            // one tcgen05.st of this thread's 16 values into TMEM lane 32 (warp mod 4) + lane
            tm_fence_after();
            uint32_t tv[32];
#pragma unroll
            for (int mf = 0; mf < MF; mf++)
#pragma unroll
                for (int nf = 0; nf < NF; nf++) {
                    const int j = 4 * (mf * NF + nf);
                    tv[j] = (uint32_t)__double2loint(acc[mf][nf][0]);
                    tv[j + 1] = (uint32_t)__double2hiint(acc[mf][nf][0]);
                    tv[j + 2] = (uint32_t)__double2loint(acc[mf][nf][1]);
                    tv[j + 3] = (uint32_t)__double2hiint(acc[mf][nf][1]);
                }
            tm_st32(tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 64 * eb + 32 * (warp >> 2), tv);
        } else {
#pragma unroll
            for (int mf = 0; mf < MF; mf++)
#pragma unroll
                for (int nf = 0; nf < NF; nf++) {
                    const int r = m0 + 8 * mf + g8, c = n0 + 8 * nf + 2 * t4;
                    reinterpret_cast<double2 *>(ebuf + eb * TILE)[r * (B / 2) + ((c >> 1) ^ eswz(r))] =
                        make_double2(acc[mf][nf][0], acc[mf][nf][1]);
                }
        }
#pragma unroll
        for (int w = MF / 2; w > 0; w >>= 1)   // fixed pairwise tree
#pragma unroll
            for (int mf = 0; mf < w; mf++) ssp[mf] += ssp[mf + w];
        ess[eb * 32 * CW + 32 * warp + lane] = ssp[0];
        if (!STORE && diag && lane == 0) etr[eb * ETR + warp] = trp;
        if constexpr (TE) {
            tm_wait_st();
            tm_fence_before();
        }
        __syncwarp();
        if (lane == 0) {
            if (warp == 0) erec[eb] = make_int4(seg, e.z, e.w, 0);
            mbar_arrive(&efull[eb]);
        }
        if (++eb == NBUF) {
            eb = 0;
            ephase ^= 1;
        }
        CLK(c_bnd += clock64() - c4;)
    }
    // end of the launch: tell the epilogue warps (once they have read the buffer's last tile)
    mbar_wait(&eempty[eb], ephase ^ 1);
    __syncwarp();
    if (lane == 0) {
        if (warp == 0) erec[eb] = make_int4(-1, 0, 0, 0);
        mbar_arrive(&efull[eb]);
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

template <int B, int CW, int WM, int WN, int STAGES, int EPI, int TA, int GRP = 0>
static spamm_status launch_gemm(spamm_ctx ctx, const GemmArgs &g, const GemmArgs &g2 = GemmArgs{})
{
    constexpr int NT = 32 * (CW + 1 + EpiCfg<B, CW>::EW);
    const size_t smem = GemmSmem<B, CW, STAGES>::bytes;
    auto kern = k_leaf_gemm<B, CW, WM, WN, STAGES, EPI, TA, GRP>;
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
    kern<<<grid, NT, smem, ctx->stream>>>(g, g2);
    CKL(ctx);
    return SPAMM_OK;
}

template <int EPI, int TA>
static spamm_status gemm_dispatch(spamm_ctx ctx, int b, const GemmArgs &g)
{
    switch (b) {
    case 64: return launch_gemm<64, 8, 2, 4, 3, EPI, TA>(ctx, g);
    case 32: return launch_gemm<32, 4, 2, 2, SPAMM_B32_STAGES, EPI, TA>(ctx, g);
    case 16: return launch_gemm<16, 1, 1, 1, 4, EPI, TA>(ctx, g);
    default: return set_err(ctx, SPAMM_EINVAL, "b=%d", b);
    }
}

static GemmArgs gemm_args(Cull *cw, spamm_mat A, spamm_mat B, const double *b_halo, spamm_mat C,
                          double *trace_part, const int32_t *seg_order, int64_t nseg, int ticket, bool device_count)
{
    if (nseg < 0) nseg = cw->nsegs;
    GemmArgs g{A->pool, B->pool, b_halo, cw->tA, cw->tB, cw->seg_code, cw->seg_start, cw->seg_len,
               (int)nseg, seg_order, C->pool, C->coord, C->slot, C->norm2 + pyr_off(C->L), trace_part,
               cw->counters + CNT_GEMM_TICKET + ticket, cw->alpha,
               device_count ? cw->counters + CNT_NSEG : nullptr, cw->peer_world, {},
               A->cap, B->cap, b_halo ? (int64_t)1 << 40 : 0, C->cap, cw->cap, cw->cap_segs, A->nb};
    for (int q = 0; q < cw->peer_world; q++) g.peer_pool[q] = cw->peer_pool[q];
    return g;
}

spamm_status gemm_run(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, const double *b_halo,
                      spamm_mat C, int epi, double *trace_part, const int32_t *seg_order, int64_t nseg,
                      int ticket, int transA, bool device_count)
{
    const GemmArgs g = gemm_args(cw, A, B, b_halo, C, trace_part, seg_order, nseg, ticket, device_count);
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

// Two plain-store products in one launch (the Y' and Z' GEMMs of a captured NS step): both
// segment counts read on the device, the launch's ticket in c1's counters.  Each segment is
// still owned by one CTA and accumulated in ascending k: results equal two launches bitwise.
spamm_status gemm_run_pair(spamm_ctx ctx, Cull *c1, spamm_mat A1, spamm_mat B1, spamm_mat C1, Cull *c2,
                           spamm_mat A2, spamm_mat B2, spamm_mat C2)
{
    if (c1->alpha != 1.0 || c2->alpha != 1.0 || c1->peer_world || c2->peer_world || A1->b != A2->b)
        return set_err(ctx, SPAMM_EINVAL, "grouped GEMM: plain single-device products of one leaf size");
    const GemmArgs g1 = gemm_args(c1, A1, B1, nullptr, C1, nullptr, nullptr, 0, 0, true);
    const GemmArgs g2 = gemm_args(c2, A2, B2, nullptr, C2, nullptr, nullptr, 0, 0, true);
    switch (A1->b) {
    case 64: return launch_gemm<64, 8, 2, 4, 3, EPI_STORE, 0, 1>(ctx, g1, g2);
    case 32: return launch_gemm<32, 4, 2, 2, SPAMM_B32_STAGES, EPI_STORE, 0, 1>(ctx, g1, g2);
    case 16: return launch_gemm<16, 1, 1, 1, 4, EPI_STORE, 0, 1>(ctx, g1, g2);
    default: return set_err(ctx, SPAMM_EINVAL, "b=%d", A1->b);
    }
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

// The captured step's fix-up in ONE launch (1 CTA): k_diag_assign's scan, then the new blocks
// filled as k_diag_fill fills them (same values, same leaf norms), then t exactly as trace_256
// forms it (threads 0..255).  At C1/C2 a launch boundary costs more than this whole kernel.
__global__ void __launch_bounds__(1024) k_diag_fix1(int32_t *slot_map, int32_t *coord, int nb, int r0, int r1,
                                                    const int32_t *base_dev, int32_t *newslot, int64_t *count_out,
                                                    int64_t cap, double *pool, int b, double value, double *leaf_n2,
                                                    const double *trace_part, double n, double *t_out)
{
    pdl_wait();
    pdl_trigger();
    __shared__ V1 sw[1024 / 32];
    __shared__ double sh[256];
    const int64_t base = *base_dev;
    int64_t run = 0;
    for (int i0 = 0; i0 < nb; i0 += 1024) {
        const int i = i0 + threadIdx.x;
        const uint32_t code = i < nb ? morton(i, i) : 0;
        V1 v{(i >= r0 && i < r1 && slot_map[code] < 0) ? 1 : 0};
        V1 tot;
        V1 ex = block_excl_scan<V1, 1024>(v, &tot, sw);
        if (i < nb) {
            const int32_t sl = v.x ? (int32_t)(base + run + ex.x) : -1;
            SPAMM_ASSERT(sl < 0 || sl < cap);
            newslot[i] = sl;
            if (v.x) {
                slot_map[code] = sl;
                coord[sl] = (int32_t)code;
            }
        }
        run += tot.x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *count_out = run;
    if (run > 0) {   // (CTA-uniform) the new diagonal blocks: value * I
        for (int i = 0; i < nb; i++) {
            const int sl = newslot[i];
            if (sl < 0) continue;
            double *d = pool + (int64_t)sl * b * b;
            for (int e = threadIdx.x; e < b * b; e += 1024) d[e] = (e / b == pool_col(e, b)) ? value : 0.0;
            if (threadIdx.x == 0) {
                double ss = 0.0;
                for (int r = 0; r < b; r++) ss += value * value;
                leaf_n2[morton(i, i)] = ss;
            }
        }
    }
    // t = (n - sum_i trace_part[i]) / n in trace_256's order
    double t = 0.0;
    if (threadIdx.x < 256)
        for (int i = threadIdx.x; i < nb; i += 256) t += trace_part[i];
    if (threadIdx.x < 256) sh[threadIdx.x] = t;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *t_out = (n - sh[0]) / n;
}

spamm_status diag_fixup_dev(spamm_ctx ctx, spamm_mat H, const int32_t *nseg_dev, double value, int32_t *newslot,
                            int64_t *dcount, const double *trace_part, double *t_out)
{
    static const int one = [] {
        const char *e = getenv("SPAMM_DIAG_ONE");
        return e && *e ? atoi(e) : 1;
    }();
    if (one && trace_part) {
        CK(launch_k(ctx, k_diag_fix1, 1, 1024, 0, H->slot, H->coord, H->nb, H->r0, H->r1, nseg_dev, newslot, dcount,
                    H->cap, H->pool, H->b, value, H->norm2 + pyr_off(H->L), trace_part, (double)H->n, t_out));
        CKL(ctx);
        return SPAMM_OK;
    }
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
