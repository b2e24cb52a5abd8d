// cull.cu — the SpAMM occlusion-cull as a level-by-level two-sided metric query.
//
// PAPER.md Eq. newspamm culls a sub-volume (i,k,j) of the product
// tensor when ||a^i|| ||b^i|| < tau ||a|| ||b||; "two-sided metric query"
// (P:329-330).  Because a child's norm never exceeds its parent's, the
// recursion returns exactly the flat leaf set
//     S = {(i,k,j) : n2A[i,k] * n2B[k,j] >= T},  T = tau^2 ||A||^2 ||B||^2
// (squared form, reading L5; absent blocks, n2 = 0, never form tasks: L3/L6).
// The GPU walks the levels breadth-first:
//   k_cull_init     level l0 = min(L,4): all 8^l0 triples in one CTA (dense start)
//   k_cull_scan     per parent task: 8-bit child mask (2 pyramid sectors read),
//                   per-quadrant child counts, single-pass decoupled look-back
//                   scan (int4) -> exclusive prefixes
//   k_cull_scatter  order-preserving compaction: children of parent group (I,J)
//                   are emitted per quadrant q = (di,dj) in (K, dk) order, so the
//                   list stays sorted by (Morton(i,j), k) with no sort; at the
//                   leaf level the groups are the output segments and tasks
//                   carry their A / B pool slots.
//   k_cull_segments compaction of segment heads -> {code, start, len}.
// Counts live in device memory; kernels are persistent / grid-stride, so the
// whole query is enqueued with no host round trip.
#include <algorithm>

#include "common.cuh"
#include "scan.cuh"

constexpr int CT = 512;  // threads per CTA of the scan kernels
constexpr int CI = 4;    // consecutive items per thread: a scan tile is CT*CI items

struct CullArgs {
    const double *a_n2, *b_n2;   // pyramids
    const int32_t *a_slot, *b_slot;
    double tau;
    int64_t cap;
    int L, r0, r1;               // leaf level; output block rows [r0, r1) (row partition, §8(e))
    int transA;                  // 1: the left operand is A^T (single channel, §8(f) f2):
                                 //    node (I,K) of A^T is node (K,I) of A, norms shared
    int counts_only;             // spamm_row_task_counts over all rows of a row-partitioned
                                 // operand: remote rows have no slots (debug check off)
};

// Morton code of node (I, K) of the left operand in A's own pyramid / slot map
__device__ __forceinline__ uint32_t a_code(const CullArgs &g, int I, int K)
{
    return g.transA ? morton(K, I) : morton(I, K);
}

// level-`lev` row index I covers leaf rows [I << (L-lev), (I+1) << (L-lev)); keep the
// sub-volume only if that range meets the local output rows
__device__ __forceinline__ bool rows_meet(const CullArgs &g, int I, int lev)
{
    const int sh = g.L - lev;
    return ((I + 1) << sh) > g.r0 && (I << sh) < g.r1;
}

__device__ __forceinline__ double cull_T(const CullArgs &g)
{
    // T = tau^2 * ||A||^2 * ||B||^2, evaluated left to right (same on every kernel)
    return ((g.tau * g.tau) * g.a_n2[0]) * g.b_n2[0];
}

__device__ __forceinline__ bool keep(double pa, double pb, double T)
{
    // strict '<' culls: survive iff pa*pb >= T; absent blocks never survive
    return pa > 0.0 && pb > 0.0 && pa * pb >= T;
}

__device__ __forceinline__ int clamp_n(const int32_t *cnt, int l, int64_t cap)
{
    int v = cnt[l];
    return v < cap ? v : (int)cap;
}

// ---------------------------------------------------------------- init
// One CTA of 1024 threads tests all 8^l0 <= 32768 candidates of level l0 (<= 32 per
// thread, consecutive), in (Morton(I,J), K) order, and writes the level-l0 records
// and counters[l0].  (Starting at l0 = 5 with <= 32 candidates per thread measured
// slower than the extra scan/scatter pair: 6.6 vs 6.0 ms of cull per C2 run.)
constexpr int INIT_L0 = 4;
// zero the counters and the look-back tile flags of all levels (a kernel rather than
// two memsets, so the whole query is one programmatic-dependent-launch chain)
// output patterns cleared by the query's first kernel (device-driven step: the slot maps
// of up to 3 matrices set to -1, their pyramids and one extra array zeroed), replacing
// memset nodes on the step's critical path
__device__ __forceinline__ void cull_clear(const CullClear &c, int64_t i0, int64_t stride)
{
    for (int m = 0; m < 3; m++) {
        if (c.slot[m])
            for (int64_t i = i0; i < c.nslot; i += stride) c.slot[m][i] = -1;
        if (c.n2[m])
            for (int64_t i = i0; i < c.nn2; i += stride) c.n2[m][i] = 0.0;
    }
    if (c.z)
        for (int64_t i = i0; i < c.nz; i += stride) c.z[i] = 0.0;
}

__global__ void k_cull_reset(int32_t *cnt, int ncnt, int32_t *flags, int64_t nflags, CullClear clr)
{
    pdl_wait();
    pdl_trigger();
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = i0; i < ncnt; i += stride) cnt[i] = 0;
    for (int64_t i = i0; i < nflags; i += stride) flags[i] = 0;
    cull_clear(clr, i0, stride);
}

// the init level for a CTA of 1024 threads (k_cull_init and k_cull_small); returns the
// level's survivor count to every thread
__device__ __forceinline__ int cull_init_body(const CullArgs &g, int l0, int4 *rec, int32_t *cnt)
{
    __shared__ V1 sw[32];
    __shared__ int gpre[(1 << (2 * INIT_L0)) + 1];   // exclusive prefix at each group (I,J) start
    const int S = 1 << l0;
    const int C = S * S * S;
    const int ipt = (C + 1023) / 1024;              // candidates per thread (<= 32)
    const double T = cull_T(g);
    const double *an = g.a_n2 + pyr_off(l0), *bn = g.b_n2 + pyr_off(l0);
    const int base = threadIdx.x * ipt;
    uint32_t f = 0;
    for (int e = 0; e < ipt; e++) {
        const int idx = base + e;
        if (idx < C) {
            const uint32_t code = idx >> l0;        // idx = code * S + K
            const int K = idx & (S - 1), I = morton_i(code), J = morton_j(code);
            if (rows_meet(g, I, l0) && keep(an[a_code(g, I, K)], bn[morton(K, J)], T)) f |= 1u << e;
        }
    }
    const int mycount = __popc(f);
    V1 vtot;
    const int ex = block_excl_scan<V1, 1024>(V1{mycount}, &vtot, sw).x;
    const int tot = vtot.x;
    for (int e = 0; e < ipt; e++) {
        const int idx = base + e;
        if (idx < C && (idx & (S - 1)) == 0) gpre[idx >> l0] = ex + __popc(f & ((1u << e) - 1u));
    }
    if (threadIdx.x == 0) gpre[S * S] = tot;
    __syncthreads();
    int run = ex;
    for (int e = 0; e < ipt; e++) {
        if (f & (1u << e)) {
            const int idx = base + e, code = idx >> l0;
            if (run < g.cap) rec[run] = make_int4(code, idx & (S - 1), gpre[code], gpre[code + 1]);
            run++;
        }
    }
    if (threadIdx.x == 0) {
        cnt[l0] = tot;
        if (tot > g.cap) cnt[CNT_OVERFLOW] = 1;
    }
    return tot;
}

__global__ void __launch_bounds__(1024) k_cull_init(CullArgs g, int l0, int4 *rec, int32_t *cnt)
{
    pdl_wait();
    pdl_trigger();
    cull_init_body(g, l0, rec, cnt);
}

// 8-bit child mask of parent record r at level l (bit 2q + dk, q = (di<<1|dj)):
//   pa = n2A_{l+1}[4*Morton(I,K) + (di<<1|dk)],  pb = n2B_{l+1}[4*Morton(K,J) + (dk<<1|dj)]
__device__ __forceinline__ uint32_t cull_parent_mask(const CullArgs &g, int l, int4 r, const double *an,
                                                     const double *bn, double T)
{
    uint32_t code = r.x;
    int K = r.y, I = morton_i(code), J = morton_j(code);
    const double2 *pa2 = reinterpret_cast<const double2 *>(an + 4 * (int64_t)a_code(g, I, K));
    const double2 *pb2 = reinterpret_cast<const double2 *>(bn + 4 * (int64_t)morton(K, J));
    double2 a01 = __ldg(pa2), a23 = __ldg(pa2 + 1), b01 = __ldg(pb2), b23 = __ldg(pb2 + 1);
    // [di][dk]; for A^T the stored child (dk, di) of node (K, I)
    double pa[2][2] = {{a01.x, a01.y}, {a23.x, a23.y}};
    if (g.transA) {
        pa[0][1] = a23.x;
        pa[1][0] = a01.y;
    }
    double pb[2][2] = {{b01.x, b01.y}, {b23.x, b23.y}};  // [dk][dj]
    uint32_t mm = 0;
#pragma unroll
    for (int di = 0; di < 2; di++) {
        if (!rows_meet(g, 2 * I + di, l + 1)) continue;
#pragma unroll
        for (int dj = 0; dj < 2; dj++)
#pragma unroll
            for (int dk = 0; dk < 2; dk++)
                if (keep(pa[di][dk], pb[dk][dj], T)) mm |= 1u << (2 * ((di << 1) | dj) + dk);
    }
    return mm;
}

__device__ __forceinline__ int4 mask_counts(uint32_t mm)
{
    return make_int4(__popc(mm & 3u), __popc((mm >> 2) & 3u), __popc((mm >> 4) & 3u), __popc((mm >> 6) & 3u));
}

// ------------------------------------------------------- level mask + scan
// Parent task t at level l -> 8 children at level l+1.  child (di,dk,dj):
//   pa = n2A_{l+1}[4*Morton(I,K) + (di<<1|dk)],  pb = n2B_{l+1}[4*Morton(K,J) + (dk<<1|dj)]
// mask bit (2q + dk), q = (di<<1|dj).
__global__ void __launch_bounds__(CT) k_cull_scan(CullArgs g, int l, const int4 *rec,
                                                  uint8_t *mask, int4 *pre, ScanTiles<int4> st,
                                                  int32_t *cnt)
{
    __shared__ int4 sw[CT / 32];
    __shared__ int s_tile;
    __shared__ int4 s_excl;
    pdl_wait();
    pdl_trigger();
    // after a capacity overflow the truncated level's group indices point past the
    // arrays: skip the rest of the query (the host grows the workspace and re-runs)
    if (__ldcg(&cnt[CNT_OVERFLOW])) return;   // written by an earlier launch: a plain L2 load
    const int n = clamp_n(cnt, l, g.cap);
    const double T = cull_T(g);
    const double *an = g.a_n2 + pyr_off(l + 1), *bn = g.b_n2 + pyr_off(l + 1);
    int tile;
    // CI consecutive parent tasks per thread: a tile is CT*CI tasks, so the
    // decoupled look-back walks CI times fewer predecessor tiles
    while ((tile = next_tile(st.ticket, n, CT * CI, &s_tile)) >= 0) {
        const int t0 = tile * (CT * CI) + threadIdx.x * CI;
        int4 c[CI];
        uint32_t m[CI];
        int4 csum = make_int4(0, 0, 0, 0);
#pragma unroll
        for (int i = 0; i < CI; i++) {
            const int t = t0 + i;
            c[i] = make_int4(0, 0, 0, 0);
            m[i] = 0;
            if (t < n) {
                const uint32_t mm = cull_parent_mask(g, l, rec[t], an, bn, T);
                m[i] = mm;
                c[i] = mask_counts(mm);
                csum = vadd(csum, c[i]);
            }
        }
        int4 tot;
        int4 ex = block_excl_scan<int4, CT>(csum, &tot, sw);
        if (threadIdx.x < 32) {
            int4 e = tile_lookback(st, tile, tot);
            if (threadIdx.x == 0) s_excl = e;
        }
        __syncthreads();
        int4 p = vadd(s_excl, ex);
#pragma unroll
        for (int i = 0; i < CI; i++) {
            const int t = t0 + i;
            if (t < n) {
                pre[t] = p;
                mask[t] = (uint8_t)m[i];
            }
            if (t == n - 1) {
                int4 e = vadd(p, c[i]);
                pre[n] = e;
                int total = e.x + e.y + e.z + e.w;
                cnt[l + 1] = total;
                if (total > g.cap) cnt[CNT_OVERFLOW] = 1;
            }
            p = vadd(p, c[i]);
        }
        __syncthreads();
    }
    if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
        pre[0] = make_int4(0, 0, 0, 0);
        cnt[l + 1] = 0;
    }
}

__device__ __forceinline__ int comp(int4 v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }

// ------------------------------------------------------------- scatter
// children of parent t, emitted per quadrant q in (K, dk) order (order-preserving)
template <bool FINAL>
__device__ __forceinline__ void cull_scatter_one(const CullArgs &g, const int4 *rec, const uint8_t *mask,
                                                 const int4 *pre, int t, int4 *rec_out, int32_t *tA, int32_t *tB,
                                                 int32_t *tK)
{
    do {
        uint32_t m = mask[t];
        if (!m) break;
        int4 r = rec[t];
        int4 P = pre[t], Ps = pre[r.z], Pe = pre[r.w];
        int base = Ps.x + Ps.y + Ps.z + Ps.w;  // children of all earlier groups
        uint32_t code = r.x;
        int K = r.y;
        int I = morton_i(code), J = morton_j(code);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            int cq = comp(Pe, q) - comp(Ps, q);
            uint32_t mq = (m >> (2 * q)) & 3u;
            if (mq) {
                int gs = base, ge = base + cq;
                int pos = base + comp(P, q) - comp(Ps, q);
#pragma unroll
                for (int dk = 0; dk < 2; dk++) {
                    if (mq & (1u << dk)) {
                        if (pos < g.cap) {
                            uint32_t ccode = 4 * code + q;
                            int ck = 2 * K + dk;
                            rec_out[pos] = make_int4((int)ccode, ck, gs, ge);
                            if (FINAL) {
                                int i = 2 * I + (q >> 1), j = 2 * J + (q & 1);
                                tA[pos] = g.a_slot[a_code(g, i, ck)];
                                tB[pos] = g.b_slot[morton(ck, j)];
                                tK[pos] = ck;
                                // a surviving triple has non-zero norms: both blocks are stored
                                // (row partition: a remote B block is -1 until the halo patch)
                                SPAMM_ASSERT(g.counts_only || (tA[pos] >= 0 && (tB[pos] >= 0 || g.r1 - g.r0 < (1 << g.L))));
                            }
                        }
                        pos++;
                    }
                }
            }
            base += cq;
        }
    } while (0);
}

template <bool FINAL>
__global__ void __launch_bounds__(256) k_cull_scatter(CullArgs g, int l, const int4 *rec,
                                                      const uint8_t *mask, const int4 *pre,
                                                      int4 *rec_out, int32_t *tA, int32_t *tB,
                                                      int32_t *tK, const int32_t *cnt)
{
    pdl_wait();
    pdl_trigger();
    if (cnt[CNT_OVERFLOW]) return;   // see k_cull_scan
    const int n = clamp_n(cnt, l, g.cap);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        cull_scatter_one<FINAL>(g, rec, mask, pre, t, rec_out, tA, tB, tK);
}

// Final records -> segments when the init level is already the leaf level.
__global__ void k_cull_leaf_direct(CullArgs g, int l, const int4 *rec, int32_t *tA, int32_t *tB,
                                   int32_t *tK, const int32_t *cnt)
{
    pdl_wait();
    pdl_trigger();
    if (cnt[CNT_OVERFLOW]) return;
    const int n = clamp_n(cnt, l, g.cap);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        int4 r = rec[t];
        int i = morton_i(r.x), j = morton_j(r.x), k = r.y;
        tA[t] = g.a_slot[a_code(g, i, k)];
        tB[t] = g.b_slot[morton(k, j)];
        tK[t] = k;
    }
}

// --------------------------------------------------------- segment heads
__global__ void __launch_bounds__(CT) k_cull_segments(const int4 *rec, int L, int64_t cap,
                                                      int64_t cap_segs, ScanTiles<V1> st,
                                                      int32_t *seg_code, int32_t *seg_start,
                                                      int32_t *seg_len, int32_t *cnt)
{
    __shared__ V1 sw[CT / 32];
    __shared__ int s_tile, s_excl;
    pdl_wait();
    if (__ldcg(&cnt[CNT_OVERFLOW])) return;   // written by an earlier launch: a plain L2 load
    const int n = clamp_n(cnt, L, cap);
    int tile;
    while ((tile = next_tile(st.ticket, n, CT * CI, &s_tile)) >= 0) {
        const int t0 = tile * (CT * CI) + threadIdx.x * CI;
        int4 r[CI];
        int hs = 0;
#pragma unroll
        for (int i = 0; i < CI; i++) {
            const int t = t0 + i;
            r[i] = make_int4(0, 0, -1, 0);
            if (t < n) r[i] = rec[t];
            hs += (t < n && r[i].z == t) ? 1 : 0;
        }
        V1 tot;
        V1 ex = block_excl_scan<V1, CT>(V1{hs}, &tot, sw);
        if (threadIdx.x < 32) {
            int e = tile_lookback(st, tile, tot).x;
            if (threadIdx.x == 0) s_excl = e;
        }
        __syncthreads();
        int s = s_excl + ex.x;
#pragma unroll
        for (int i = 0; i < CI; i++) {
            const int t = t0 + i;
            const int h = (t < n && r[i].z == t) ? 1 : 0;
            if (h && s < cap_segs) {
                seg_code[s] = r[i].x;
                seg_start[s] = t;
                seg_len[s] = r[i].w - r[i].z;
            }
            if (t == n - 1) {
                cnt[CNT_NSEG] = s + h;
                if (s + h > cap_segs) cnt[CNT_OVERFLOW] = 1;
            }
            s += h;
        }
        __syncthreads();
    }
    if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) cnt[CNT_NSEG] = 0;
}

// ------------------------------------------------------- single-CTA query
// Small problems (the level sizes of C1/C2 are ~10^2-10^4 triples) are latency-bound:
// the multi-kernel chain costs ~9 launches per product.  k_cull_small runs the SAME
// algorithm -- init level, then per level the child masks, the int4 exclusive scan of
// per-quadrant counts (sequential tiles of one CTA instead of a decoupled look-back
// across CTAs), the order-preserving scatter, and the segment compaction -- in one
// 1024-thread CTA with block barriers between phases.  Every array it writes equals
// the chain's bit for bit (same records, prefixes, tasks, segments; same overflow
// rule), so the products do not depend on which form ran.
constexpr int SMALL_T = 1024;

// a level of up to SMALL_STAGE parents keeps its prefixes and masks in shared memory, so
// the scatter's reads of pre[t], pre[r.z], pre[r.w] and mask[t] are not global round trips
constexpr int SMALL_STAGE = 8191;
constexpr size_t SMALL_SMEM = (SMALL_STAGE + 1) * sizeof(int4) + (SMALL_STAGE + 1);

__global__ void __launch_bounds__(SMALL_T) k_cull_small(CullArgs g, int l0, int4 *rec0, int4 *rec1, uint8_t *mask_g,
                                                        int4 *pre_g, int32_t *tA, int32_t *tB, int32_t *tK,
                                                        int64_t cap_segs, int32_t *seg_code, int32_t *seg_start,
                                                        int32_t *seg_len, int32_t *cnt, CullClear clr)
{
    __shared__ int4 sw4[SMALL_T / 32];
    __shared__ V1 sw1[SMALL_T / 32];
    extern __shared__ __align__(16) unsigned char small_smem[];
    int4 *const pre_s = reinterpret_cast<int4 *>(small_smem);
    uint8_t *const mask_s = small_smem + (SMALL_STAGE + 1) * sizeof(int4);
    pdl_wait();
    pdl_trigger();
    for (int i = threadIdx.x; i < 64; i += SMALL_T) cnt[i] = 0;
    cull_clear(clr, threadIdx.x, SMALL_T);
    __syncthreads();
    int4 *rec[2] = {rec0, rec1};
    int cur = 0;
    // every thread holds each level's count (the scan totals are block-wide), so neither
    // the count nor the overflow flag (set exactly when a count exceeds cap; the counters
    // were zeroed above) is re-read from global memory between phases
    int nl = cull_init_body(g, l0, rec[cur], cnt);
    __syncthreads();
    const double T = cull_T(g);
    for (int l = l0; l < g.L; l++) {
        if (nl > g.cap) return;
        const int n = nl;
        const double *an = g.a_n2 + pyr_off(l + 1), *bn = g.b_n2 + pyr_off(l + 1);
        const bool staged = n <= SMALL_STAGE;
        int4 *const pre = staged ? pre_s : pre_g;
        uint8_t *const mask = staged ? mask_s : mask_g;
        // masks + per-quadrant counts, exclusive int4 scan in task order
        int4 carry = make_int4(0, 0, 0, 0);
        for (int t0 = 0; t0 < n; t0 += SMALL_T * CI) {
            const int tb = t0 + threadIdx.x * CI;
            int4 c[CI];
            uint32_t m[CI];
            int4 csum = make_int4(0, 0, 0, 0);
#pragma unroll
            for (int i = 0; i < CI; i++) {
                const int t = tb + i;
                m[i] = t < n ? cull_parent_mask(g, l, rec[cur][t], an, bn, T) : 0u;
                c[i] = mask_counts(m[i]);
                csum = vadd(csum, c[i]);
            }
            int4 tot;
            int4 p = vadd(carry, block_excl_scan<int4, SMALL_T>(csum, &tot, sw4));
#pragma unroll
            for (int i = 0; i < CI; i++) {
                const int t = tb + i;
                if (t < n) {
                    pre[t] = p;
                    mask[t] = (uint8_t)m[i];
                }
                p = vadd(p, c[i]);
            }
            carry = vadd(carry, tot);
        }
        const int total = carry.x + carry.y + carry.z + carry.w;
        if (threadIdx.x == 0) {
            pre[n] = carry;
            cnt[l + 1] = total;
            if (total > g.cap) cnt[CNT_OVERFLOW] = 1;
        }
        __syncthreads();
        if (total > g.cap) return;
        if (l + 1 == g.L) {
            for (int t = threadIdx.x; t < n; t += SMALL_T)
                cull_scatter_one<true>(g, rec[cur], mask, pre, t, rec[cur ^ 1], tA, tB, tK);
        } else {
            for (int t = threadIdx.x; t < n; t += SMALL_T)
                cull_scatter_one<false>(g, rec[cur], mask, pre, t, rec[cur ^ 1], nullptr, nullptr, nullptr);
        }
        cur ^= 1;
        nl = total;
        __syncthreads();
    }
    if (nl > g.cap) return;
    const int n = nl;
    if (l0 == g.L) {   // the init level is the leaf level: tasks straight from the records
        for (int t = threadIdx.x; t < n; t += SMALL_T) {
            const int4 r = rec[cur][t];
            const int i = morton_i(r.x), j = morton_j(r.x), k = r.y;
            tA[t] = g.a_slot[a_code(g, i, k)];
            tB[t] = g.b_slot[morton(k, j)];
            tK[t] = k;
        }
    }
    // segment heads (record r starts its group: r.z == t) -> {code, start, len}
    int carry = 0;
    for (int t0 = 0; t0 < n; t0 += SMALL_T * CI) {
        const int tb = t0 + threadIdx.x * CI;
        int4 r[CI];
        int hs = 0;
#pragma unroll
        for (int i = 0; i < CI; i++) {
            const int t = tb + i;
            r[i] = t < n ? rec[cur][t] : make_int4(0, 0, -1, 0);
            hs += (t < n && r[i].z == t) ? 1 : 0;
        }
        V1 tot;
        int sidx = carry + block_excl_scan<V1, SMALL_T>(V1{hs}, &tot, sw1).x;
#pragma unroll
        for (int i = 0; i < CI; i++) {
            const int t = tb + i;
            if (t < n && r[i].z == t) {
                if (sidx < cap_segs) {
                    seg_code[sidx] = r[i].x;
                    seg_start[sidx] = t;
                    seg_len[sidx] = r[i].w - r[i].z;
                }
                sidx++;
            }
        }
        carry += tot.x;
    }
    if (threadIdx.x == 0) {
        cnt[CNT_NSEG] = carry;
        if (carry > cap_segs) cnt[CNT_OVERFLOW] = 1;
    }
}

// ------------------------------------------------------- flat small query
// For nb <= 128 the whole query is cheaper as a flat test than as a walk: the walk's levels
// are a chain of dependent global round trips (k_cull_small: ~40 us per product at C2,
// 1 CTA), while all nb^3 <= 2.1M leaf triples, and the 8^l triples of each level above, can
// be tested at once on every SM.  Because a parent's n2 is >= each child's (sums of
// non-negative numbers, rounded monotonically) and rounded products are monotone, a triple
// passes the test at level l exactly when the walk reaches and keeps it: the walk's
// survivors at level l are the level-l triples that pass, and its leaf tasks are the
// passing leaf triples.  Three launches write exactly what the walk writes (level counts,
// the final records {Morton(i,j), k, group start, group end}, tA/tB/tK in (Morton(i,j), k)
// order, segments, NSEG, overflow):
//   k_cullf_count (grid)  tiles of 8 x 8 output pairs (i,j) (Morton code m), their leaf norms
//                         staged in shared memory; one warp per pair: ballots of the k that
//                         pass -> pmask[m][w], count -> pcnt[m]; per-CTA counts of the passing
//                         triples of each level l0..L-1 -> lvl[l][cta]
//   k_cullf_scan (1 CTA)  level counts, exclusive scan of (tasks, non-empty) over m ->
//                         ppre[m] = (first task, segment), totals, overflow
//   k_cullf_emit (grid)   one warp per non-empty pair: its segment, records and tasks
// (tests/test_gpu_determinism.py: SPAMM_CULL_FLAT=0/1 give the same NS runs bitwise, every
// product's task, segment and per-level survivor counts included)
constexpr int FLAT_T = 256;

__global__ void __launch_bounds__(FLAT_T) k_cullf_count(CullArgs g, int l0, uint32_t *pmask, int32_t *pcnt,
                                                        int32_t *lvl, CullClear clr)
{
    pdl_wait();
    pdl_trigger();
    __shared__ int sred[FLAT_T / 32];
    const int nbL = 1 << g.L, W = (nbL + 31) >> 5;
    const int64_t gtid = blockIdx.x * (int64_t)FLAT_T + threadIdx.x, gstride = (int64_t)gridDim.x * FLAT_T;
    cull_clear(clr, gtid, gstride);
    const double T = cull_T(g);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        // leaf pairs in tiles of TI x TI: the TI rows of A's leaf norms and TI columns of B's
        // (each a run of TI x TI Morton quadtree nodes: contiguous) staged in shared memory
        __shared__ double sA[8 * 128], sB[8 * 128];
        const double *an = g.a_n2 + pyr_off(g.L), *bn = g.b_n2 + pyr_off(g.L);
        const int TI = nbL < 8 ? nbL : 8, tpr = nbL / TI;
        for (int tile = blockIdx.x; tile < tpr * tpr; tile += gridDim.x) {
            const int i0 = (tile / tpr) * TI, j0 = (tile % tpr) * TI;
            __syncthreads();
            for (int e = threadIdx.x; e < TI * nbL; e += FLAT_T) {
                const int r = e / nbL, k = e % nbL;
                sA[e] = an[a_code(g, i0 + r, k)];
                sB[e] = bn[morton(k, j0 + r)];
            }
            __syncthreads();
            for (int q = warp; q < TI * TI; q += FLAT_T / 32) {
                const int ri = q / TI, rj = q % TI, i = i0 + ri, j = j0 + rj;
                const uint32_t m = morton(i, j);
                const bool rm = rows_meet(g, i, g.L);
                int c = 0;
                for (int w = 0; w < W; w++) {
                    const int k = 32 * w + lane;
                    const bool kp = rm && k < nbL && keep(sA[ri * nbL + k], sB[rj * nbL + k], T);
                    const uint32_t bal = __ballot_sync(0xffffffffu, kp);
                    if (lane == 0) pmask[(int64_t)m * W + w] = bal;
                    c += __popc(bal);
                }
                if (lane == 0) pcnt[m] = c;
            }
        }
    }
    for (int l = l0; l < g.L; l++) {
        const int S = 1 << l;
        const int64_t C = (int64_t)S * S * S;
        const double *an = g.a_n2 + pyr_off(l), *bn = g.b_n2 + pyr_off(l);
        int c = 0;
        for (int64_t idx = gtid; idx < C; idx += gstride) {
            const uint32_t code = (uint32_t)(idx / S);
            const int K = (int)(idx % S), I = morton_i(code), J = morton_j(code);
            if (rows_meet(g, I, l) && keep(an[a_code(g, I, K)], bn[morton(K, J)], T)) c++;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) sred[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < FLAT_T / 32; w++) t += sred[w];
            lvl[(l - l0) * gridDim.x + blockIdx.x] = t;
        }
        __syncthreads();
    }
}

// (every count is an integer: the reductions' order does not matter).  The nb^2 <= 16384
// counts go through shared memory (coalesced global loads and stores, conflict-free warp
// scans: a per-thread run of consecutive pairs had 16-way bank conflicts, 23 us per launch).
constexpr int FLAT_PT = 16;
constexpr size_t FLAT_SMEM = sizeof(int32_t) * 3 * SMALL_T * FLAT_PT;   // counts, prefixes, segment ids
__global__ void __launch_bounds__(SMALL_T) k_cullf_scan(CullArgs g, int l0, const int32_t *pcnt, int2 *ppre,
                                                        const int32_t *lvl, int nlvl_cta, int64_t cap_segs,
                                                        int32_t *cnt)
{
    __shared__ int4 sw4[SMALL_T / 32];
    __shared__ int sred[SMALL_T / 32];
    extern __shared__ int32_t fsm[];
    int32_t *sn = fsm, *sp = fsm + SMALL_T * FLAT_PT, *ss = sp + SMALL_T * FLAT_PT;
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 64; i += SMALL_T) cnt[i] = 0;
    const int np = 1 << (2 * g.L), pt = (np + SMALL_T - 1) / SMALL_T;
    for (int m = tid; m < np; m += SMALL_T) sn[m] = pcnt[m];
    // level counts: the per-CTA partials summed by the whole CTA
    for (int li = 0; li < g.L - l0; li++) {
        int t = 0;
        for (int c = tid; c < nlvl_cta; c += SMALL_T) t += lvl[li * nlvl_cta + c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) sred[warp] = t;
        __syncthreads();
        if (tid == 0) {
            int u = 0;
            for (int w = 0; w < SMALL_T / 32; w++) u += sred[w];
            cnt[l0 + li] = u;
            if (u > g.cap) cnt[CNT_OVERFLOW] = 1;
        }
        __syncthreads();
    }
    __syncthreads();
    // warp w scans the pairs [w*32*pt, (w+1)*32*pt) in pt rounds of 32 (lane = pair within the
    // round: conflict-free shared-memory access), after a block scan of the warp totals
    const int base = warp * 32 * pt;
    int2 ws = make_int2(0, 0);
    for (int i = 0; i < pt; i++) {
        const int e = base + 32 * i + lane, v = e < np ? sn[e] : 0;
        ws.x += v;
        ws.y += v > 0 ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ws.x += __shfl_xor_sync(0xffffffffu, ws.x, o);
        ws.y += __shfl_xor_sync(0xffffffffu, ws.y, o);
    }
    if (lane == 0) sw4[warp] = make_int4(ws.x, ws.y, 0, 0);
    __syncthreads();
    int2 run = make_int2(0, 0), tot = make_int2(0, 0);
    for (int w = 0; w < SMALL_T / 32; w++) {
        if (w < warp) run = make_int2(run.x + sw4[w].x, run.y + sw4[w].y);
        tot = make_int2(tot.x + sw4[w].x, tot.y + sw4[w].y);
    }
    for (int i = 0; i < pt; i++) {
        const int e = base + 32 * i + lane, v = e < np ? sn[e] : 0;
        int2 inc = make_int2(v, v > 0 ? 1 : 0);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int ox = __shfl_up_sync(0xffffffffu, inc.x, d), oy = __shfl_up_sync(0xffffffffu, inc.y, d);
            if (lane >= d) {
                inc.x += ox;
                inc.y += oy;
            }
        }
        if (e < np) {
            sp[e] = run.x + inc.x - v;
            ss[e] = run.y + inc.y - (v > 0 ? 1 : 0);
        }
        run.x += __shfl_sync(0xffffffffu, inc.x, 31);
        run.y += __shfl_sync(0xffffffffu, inc.y, 31);
    }
    __syncthreads();
    for (int m = tid; m < np; m += SMALL_T) ppre[m] = make_int2(sp[m], ss[m]);
    if (tid == 0) {
        cnt[g.L] = tot.x;
        cnt[CNT_NSEG] = tot.y;
        if (tot.x > g.cap || tot.y > cap_segs) cnt[CNT_OVERFLOW] = 1;
    }
}

__global__ void __launch_bounds__(FLAT_T) k_cullf_emit(CullArgs g, const uint32_t *pmask, const int32_t *pcnt,
                                                       const int2 *ppre,
                                                       int4 *rec, int32_t *tA, int32_t *tB, int32_t *tK,
                                                       int32_t *seg_code, int32_t *seg_start, int32_t *seg_len,
                                                       const int32_t *cnt)
{
    pdl_wait();
    pdl_trigger();
    if (cnt[CNT_OVERFLOW]) return;
    const int nbL = 1 << g.L, W = (nbL + 31) >> 5, lane = threadIdx.x & 31;
    const int64_t gtid = blockIdx.x * (int64_t)FLAT_T + threadIdx.x, gstride = (int64_t)gridDim.x * FLAT_T;
    const int nw = (int)(gstride >> 5), np = nbL * nbL;
    // chunks of 32 pairs per warp: lane l looks at pair m0 + l, then the warp emits the
    // non-empty ones in order
    for (int m0 = (int)(gtid >> 5) * 32; m0 < np; m0 += nw * 32) {
        const int ml = m0 + lane, cl = ml < np ? pcnt[ml] : 0;
        const int2 pl = ml < np ? ppre[ml] : make_int2(0, 0);
        uint32_t todo = __ballot_sync(0xffffffffu, cl > 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int m = m0 + src, c = __shfl_sync(0xffffffffu, cl, src);
            const int px = __shfl_sync(0xffffffffu, pl.x, src), py = __shfl_sync(0xffffffffu, pl.y, src);
            const int i = morton_i((uint32_t)m), j = morton_j((uint32_t)m);
            const int gs = px, ge = px + c;
            if (lane == 0) {
                seg_code[py] = m;
                seg_start[py] = gs;
                seg_len[py] = c;
            }
            int run = gs;
            for (int w = 0; w < W; w++) {
                const uint32_t bal = pmask[(int64_t)m * W + w];
                if ((bal >> lane) & 1u) {
                    const int k = 32 * w + lane, pos = run + __popc(bal & ((1u << lane) - 1u));
                    rec[pos] = make_int4(m, k, gs, ge);
                    tA[pos] = g.a_slot[a_code(g, i, k)];
                    tB[pos] = g.b_slot[morton(k, j)];
                    tK[pos] = k;
                    SPAMM_ASSERT(g.counts_only || (tA[pos] >= 0 && (tB[pos] >= 0 || g.r1 - g.r0 < (1 << g.L))));
                }
                run += __popc(bal);
            }
        }
    }
}

// ------------------------------------------------------------- host side
void cull_free(spamm_ctx ctx, Cull *cw)
{
    if (!cw) return;
    int64_t cap = cw->cap, cs = cw->cap_segs, tiles = cw->tiles;
    dev_free(ctx, cw->rec[0], sizeof(int4) * cap);
    dev_free(ctx, cw->rec[1], sizeof(int4) * cap);
    dev_free(ctx, cw->pre, sizeof(int4) * (cap + 1));
    dev_free(ctx, cw->mask, cap);
    dev_free(ctx, cw->tA, sizeof(int32_t) * cap);
    dev_free(ctx, cw->tB, sizeof(int32_t) * cap);
    dev_free(ctx, cw->tK, sizeof(int32_t) * cap);
    dev_free(ctx, cw->seg_code, sizeof(int32_t) * cs);
    dev_free(ctx, cw->seg_start, sizeof(int32_t) * cs);
    dev_free(ctx, cw->seg_len, sizeof(int32_t) * cs);
    dev_free(ctx, cw->tile_flag, sizeof(int32_t) * (SPAMM_MAX_L + 2) * tiles);
    dev_free(ctx, cw->tile_agg, sizeof(int4) * tiles);
    dev_free(ctx, cw->tile_pre, sizeof(int4) * tiles);
    cw->rec[0] = cw->rec[1] = cw->pre = cw->tile_agg = cw->tile_pre = nullptr;
    cw->mask = nullptr;
    cw->tA = cw->tB = cw->tK = cw->seg_code = cw->seg_start = cw->seg_len = cw->tile_flag = nullptr;
    cw->cap = cw->cap_segs = cw->tiles = 0;
}

static spamm_status cull_alloc(spamm_ctx ctx, Cull *cw, int64_t cap, int64_t cap_segs)
{
    cull_free(ctx, cw);
    cw->gen++;
    cw->cap = cap;
    cw->cap_segs = cap_segs;
    cw->tiles = cdiv(cap + 1, CT * CI);
    cw->rec[0] = dalloc<int4>(ctx, cap);
    cw->rec[1] = dalloc<int4>(ctx, cap);
    cw->pre = dalloc<int4>(ctx, cap + 1);
    cw->mask = dalloc<uint8_t>(ctx, cap);
    cw->tA = dalloc<int32_t>(ctx, cap);
    cw->tB = dalloc<int32_t>(ctx, cap);
    cw->tK = dalloc<int32_t>(ctx, cap);
    cw->seg_code = dalloc<int32_t>(ctx, cap_segs);
    cw->seg_start = dalloc<int32_t>(ctx, cap_segs);
    cw->seg_len = dalloc<int32_t>(ctx, cap_segs);
    cw->tile_flag = dalloc<int32_t>(ctx, (SPAMM_MAX_L + 2) * cw->tiles);
    cw->tile_agg = dalloc<int4>(ctx, cw->tiles);
    cw->tile_pre = dalloc<int4>(ctx, cw->tiles);
    if (!cw->counters) {
        cw->counters = dalloc<int32_t>(ctx, 64);
        if (cudaMallocHost(&cw->hcnt, sizeof(int32_t) * 64) != cudaSuccess) cw->hcnt = nullptr;
    }
    if (!cw->rec[0] || !cw->rec[1] || !cw->pre || !cw->mask || !cw->tA || !cw->tB || !cw->tK ||
        !cw->seg_code || !cw->seg_start || !cw->seg_len || !cw->tile_flag || !cw->tile_agg ||
        !cw->tile_pre || !cw->counters || !cw->hcnt)
        return set_err(ctx, SPAMM_ENOMEM, "cull workspace (%lld tasks)", (long long)cap);
    return SPAMM_OK;
}

// The single-CTA query for small problems: nb <= 128 (C1, C2), decided from the shape
// alone so a captured graph and the host-driven path always agree.
// SPAMM_CULL_SMALL=0 disables it (A/B checks).
static bool cull_small_ok(spamm_ctx ctx, const Cull *cw, spamm_mat A)
{
    static const int mode = [] {
        const char *e = getenv("SPAMM_CULL_SMALL");
        return e && *e ? atoi(e) : 1;
    }();
    if (!mode) return false;
    if (A->nb <= 128) return true;
    (void)ctx;
    return false;
}

// The flat query (nb <= 128; SPAMM_CULL_FLAT=1 selects it, default off: measured slower than
// the single-CTA walk — C2 6.89 vs 6.63 ms, C1 2.26 vs 1.99 ms per run; under ncu its three
// launches take 14 + 14 + 18 us per product against the walk's 41 us in one, and in the
// step the extra launch gaps cost more than the shorter chain saves) needs the workspace to hold the
// nb^2 pair records (rec[1]), their pass masks (pre) and the per-CTA level counts (mask);
// decided from the shape and the capacity alone (the host-driven and the captured step
// always size the workspace for at least nb^2 records at these sizes).
static bool cull_flat_ok(spamm_ctx ctx, const Cull *cw, spamm_mat A)
{
    static const int mode = [] {
        const char *e = getenv("SPAMM_CULL_FLAT");
        return e && *e ? atoi(e) : 0;
    }();
    if (!mode || A->nb > 128) return false;
    const int64_t np = (int64_t)A->nb * A->nb, W = (A->nb + 31) / 32;
    const int l0 = A->L < INIT_L0 ? A->L : INIT_L0;
    const int64_t lvl_bytes = (int64_t)sizeof(int32_t) * (A->L - l0) * 4 * ctx->sm_count;
    return cw->cap >= np && 4 * (cw->cap + 1) >= np * W && cw->cap >= lvl_bytes;
}

// Enqueue the whole query (no host sync).
static spamm_status cull_enqueue(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int r0,
                                 int r1, int transA, const CullClear *clear = nullptr)
{
    const CullClear clr = clear ? *clear : CullClear{};
    const int L = A->L;
    const int l0 = L < INIT_L0 ? L : INIT_L0;
    cw->L = L;
    cw->l0 = l0;
    cw->b = A->b;
    CullArgs g{A->norm2, B->norm2, A->slot, B->slot, tau, cw->cap, L, r0, r1, transA, cw->counts_only ? 1 : 0};
    cudaStream_t s = ctx->stream;
    if (cull_flat_ok(ctx, cw, A)) {
        // pair records in rec[1], the pass masks in pre, per-CTA level counts in mask
        const int64_t np = (int64_t)A->nb * A->nb;
        const int ti = A->nb < 8 ? A->nb : 8;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(np / (ti * ti), 4 * ctx->sm_count));
        cw->final_buf = 0;
        int32_t *pcnt = reinterpret_cast<int32_t *>(cw->rec[1]);      // [np] counts, then
        int2 *ppre = reinterpret_cast<int2 *>(pcnt + (np + 1) / 2 * 2);   // [np] (first task, segment)
        uint32_t *pmask = reinterpret_cast<uint32_t *>(cw->pre);
        int32_t *lvl = reinterpret_cast<int32_t *>(cw->mask);
        static std::atomic<uint64_t> configured{0};
        CK(once_per_device(configured, ctx->device, [&]() {
            return cudaFuncSetAttribute(k_cullf_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FLAT_SMEM);
        }));
        CK(launch_k(ctx, k_cullf_count, grid, FLAT_T, 0, g, l0, pmask, pcnt, lvl, clr));
        CKL(ctx);
        CK(launch_k(ctx, k_cullf_scan, 1, SMALL_T, FLAT_SMEM, g, l0, (const int32_t *)pcnt, ppre, (const int32_t *)lvl,
                    grid, cw->cap_segs, cw->counters));
        CKL(ctx);
        CK(launch_k(ctx, k_cullf_emit, grid, FLAT_T, 0, g, (const uint32_t *)pmask, (const int32_t *)pcnt,
                    (const int2 *)ppre, cw->rec[0], cw->tA, cw->tB, cw->tK, cw->seg_code, cw->seg_start, cw->seg_len,
                    (const int32_t *)cw->counters));
        CKL(ctx);
        return SPAMM_OK;
    }
    if (cull_small_ok(ctx, cw, A)) {
        cw->final_buf = (L - l0) & 1;
        static std::atomic<uint64_t> configured{0};
        CK(once_per_device(configured, ctx->device, [&]() {
            return cudaFuncSetAttribute(k_cull_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMALL_SMEM);
        }));
        CK(launch_k(ctx, k_cull_small, 1, SMALL_T, SMALL_SMEM, g, l0, cw->rec[0], cw->rec[1], cw->mask, cw->pre, cw->tA,
                    cw->tB, cw->tK, cw->cap_segs, cw->seg_code, cw->seg_start, cw->seg_len, cw->counters, clr));
        CKL(ctx);
        return SPAMM_OK;
    }
    const int64_t nflags = (int64_t)(SPAMM_MAX_L + 2) * cw->tiles;
    const int pdl = A->dist ? 0 : 1;   // row partition: the predecessor may be a collective
    if (pdl) {
        const int64_t work = std::max<int64_t>(nflags, std::max(clr.nslot, clr.nn2));
        CK(launch_pdl(k_cull_reset, (int)std::min<int64_t>(cdiv(work, 256), 4 * ctx->sm_count), 256, 0, s,
                      cw->counters, 64, cw->tile_flag, nflags, clr));
        CKL(ctx);
    } else {
        if (clear) return set_err(ctx, SPAMM_EINVAL, "pattern clearing needs the single-device query");
        CK(cudaMemsetAsync(cw->counters, 0, sizeof(int32_t) * 64, s));
        CK(cudaMemsetAsync(cw->tile_flag, 0, sizeof(int32_t) * nflags, s));
    }
    int cur = 0;
    if (pdl) CK(launch_pdl(k_cull_init, 1, 1024, 0, s, g, l0, cw->rec[cur], cw->counters));
    else k_cull_init<<<1, 1024, 0, s>>>(g, l0, cw->rec[cur], cw->counters);
    CKL(ctx);
    const int persist = 2 * ctx->sm_count;
    // grids sized from the previous query's level counts (+25 %), else the capacity
    const bool have_prev = cw->prevL == L && !ctx->capturing;
    auto expect = [&](int l) -> int64_t {
        return have_prev ? (int64_t)cw->prev[l] + cw->prev[l] / 4 + 1 : cw->cap;
    };
    auto scan_grid = [&](int l) -> int {
        const int64_t t = cdiv(expect(l), (int64_t)CT * CI);
        return (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(t, cw->tiles), persist));
    };
    auto flat_grid = [&](int l) -> int {
        return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(std::min(expect(l), cw->cap), 256),
                                                            4 * ctx->sm_count));
    };
    for (int l = l0; l < L; l++) {
        ScanTiles<int4> st{cw->tile_flag + (int64_t)(l - l0) * cw->tiles, cw->tile_agg, cw->tile_pre,
                           cw->counters + CNT_TICKET + l};
        CK(launch_pdl(k_cull_scan, scan_grid(l), CT, 0, s, g, l, cw->rec[cur], cw->mask, cw->pre, st, cw->counters));
        CKL(ctx);
        if (l + 1 == L)
            CK(launch_pdl(k_cull_scatter<true>, flat_grid(l), 256, 0, s, g, l, cw->rec[cur], cw->mask, cw->pre,
                          cw->rec[cur ^ 1], cw->tA, cw->tB, cw->tK, cw->counters));
        else
            CK(launch_pdl(k_cull_scatter<false>, flat_grid(l), 256, 0, s, g, l, cw->rec[cur], cw->mask, cw->pre,
                          cw->rec[cur ^ 1], (int32_t *)nullptr, (int32_t *)nullptr, (int32_t *)nullptr,
                          cw->counters));
        CKL(ctx);
        cur ^= 1;
    }
    if (l0 == L) {
        CK(launch_pdl(k_cull_leaf_direct, flat_grid(L), 256, 0, s, g, L, cw->rec[cur], cw->tA, cw->tB, cw->tK,
                      cw->counters));
        CKL(ctx);
    }
    cw->final_buf = cur;
    ScanTiles<V1> st{cw->tile_flag + (int64_t)(SPAMM_MAX_L + 1) * cw->tiles, (V1 *)cw->tile_agg,
                     (V1 *)cw->tile_pre, cw->counters + CNT_TICKET + SPAMM_MAX_L + 1};
    CK(launch_pdl(k_cull_segments, scan_grid(L), CT, 0, s, cw->rec[cur], L, cw->cap, cw->cap_segs, st, cw->seg_code,
                  cw->seg_start, cw->seg_len, cw->counters));
    CKL(ctx);
    return SPAMM_OK;
}

// the pattern clearing of a captured step as a kernel of its own (on any stream), so it can
// run beside the X cull instead of inside it (one CTA clearing ~0.7 MB at C2)
spamm_status cull_clear_enqueue(spamm_ctx ctx, const CullClear &clr)
{
    const int64_t work = std::max<int64_t>(std::max(clr.nslot, clr.nn2), clr.nz);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(work, 256), 2 * ctx->sm_count));
    k_cull_reset<<<grid, 256, 0, ctx->stream>>>(nullptr, 0, nullptr, 0, clr);
    CKL(ctx);
    return SPAMM_OK;
}

spamm_status cull_enqueue_fixed(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau,
                                const CullClear *clear)
{
    return cull_enqueue(ctx, cw, A, B, tau, 0, A->nb, 0, clear);
}

spamm_status cull_reserve(spamm_ctx ctx, Cull *cw, int64_t cap, int64_t cap_segs)
{
    if (cw->tA && cw->cap >= cap && cw->cap_segs >= cap_segs) return SPAMM_OK;
    ST(cull_alloc(ctx, cw, std::max(cap, cw->cap), std::max(cap_segs, cw->cap_segs)));
    if (cw->hint < cw->cap) cw->hint = cw->cap;
    return SPAMM_OK;
}

// counts of a query that did not overflow -> host state, stats, next capacity hint
static void cull_accept(spamm_ctx ctx, Cull *cw)
{
    cw->ntasks = cw->hcnt[cw->L];
    cw->nsegs = cw->hcnt[CNT_NSEG];
    spamm_stats &s = cw->stats;
    s = spamm_stats{};
    s.tasks = cw->ntasks;
    s.segments = cw->nsegs;
    for (int l = cw->l0; l <= cw->L && l < 24; l++) s.level_survivors[l] = cw->hcnt[l];
    s.candidates = cw->L > cw->l0 ? 8 * (int64_t)cw->hcnt[cw->L - 1] : ((int64_t)1 << (3 * cw->L));
    s.flops = 2.0 * (double)cw->b * cw->b * cw->b * (double)cw->ntasks;
    cw->prevL = cw->L;
    for (int l = 0; l <= cw->L && l < SPAMM_MAX_L + 2; l++) cw->prev[l] = l >= cw->l0 ? cw->hcnt[l] : 0;
    // next capacity hint: 25% headroom over the largest level seen
    int64_t mx = 0;
    for (int l = cw->l0; l <= cw->L; l++) mx = cw->hcnt[l] > mx ? cw->hcnt[l] : mx;
    int64_t h = mx + mx / 4 + 1024;
    if (h > cw->hint) cw->hint = h;
    ctx->last = cw;
}

static spamm_status cull_ensure(spamm_ctx ctx, Cull *cw, spamm_mat A)
{
    int64_t nb = A->nb;
    int64_t want = cw->hint > 0 ? cw->hint : (int64_t)1 << 16;
    if (want > cw->cap || cw->cap_segs < nb * nb || !cw->tA) {
        int64_t cap = want > cw->cap ? want : cw->cap;
        ST(cull_alloc(ctx, cw, cap, nb * nb));
    }
    return SPAMM_OK;
}

// Split form for batching several queries behind one host round trip: cull_start
// enqueues, the caller fetches cw->counters into cw->hcnt (with other small values),
// cull_complete accepts the counts or, after an overflow, grows and re-runs.
spamm_status cull_start(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int r0, int r1, int transA)
{
    ST(cull_ensure(ctx, cw, A));
    return cull_enqueue(ctx, cw, A, B, tau, r0, r1, transA);
}

spamm_status cull_complete(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int r0, int r1,
                           int transA)
{
    if (!cw->hcnt[CNT_OVERFLOW]) {
        cull_accept(ctx, cw);
        return SPAMM_OK;
    }
    return cull_run(ctx, cw, A, B, tau, r0, r1, transA);
}

spamm_status cull_run(spamm_ctx ctx, Cull *cw, spamm_mat A, spamm_mat B, double tau, int r0, int r1, int transA)
{
    const int64_t nb = A->nb;
    ST(cull_ensure(ctx, cw, A));
    for (int attempt = 0; attempt < 8; attempt++) {
        ST(cull_enqueue(ctx, cw, A, B, tau, r0, r1, transA));
        ST(fetch1(ctx, cw->counters, cw->hcnt, sizeof(int32_t) * 64));
        if (!cw->hcnt[CNT_OVERFLOW]) {
            cull_accept(ctx, cw);
            return SPAMM_OK;
        }
        // grow: the largest count seen (the first overflowing level) times 2
        int64_t mx = cw->cap;
        for (int l = cw->l0; l <= cw->L; l++) mx = cw->hcnt[l] > mx ? cw->hcnt[l] : mx;
        int64_t cap = 2 * mx;
        if (cap > ((int64_t)1 << 30)) return set_err(ctx, SPAMM_ECAPACITY, "cull capacity > 2^30 tasks");
        ST(cull_alloc(ctx, cw, cap, nb * nb));
        cw->hint = cap;
    }
    return set_err(ctx, SPAMM_ECAPACITY, "cull capacity did not converge");
}

spamm_status cull_export(spamm_ctx ctx, Cull *cw, int32_t *ikj, int64_t cap, int64_t *n)
{
    *n = cw->ntasks;
    int64_t m = cw->ntasks < cap ? cw->ntasks : cap;
    if (m <= 0) return SPAMM_OK;
    int4 *h = nullptr;
    CK(cudaMallocHost(&h, sizeof(int4) * m));
    cudaError_t e = cudaMemcpyAsync(h, cw->rec[cw->final_buf], sizeof(int4) * m, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        cudaFreeHost(h);
        return check_cuda(ctx, e, "task export");
    }
    for (int64_t t = 0; t < m; t++) {
        uint32_t code = h[t].x;
        ikj[3 * t + 0] = (int32_t)morton_i(code);
        ikj[3 * t + 1] = h[t].y;
        ikj[3 * t + 2] = (int32_t)morton_j(code);
    }
    cudaFreeHost(h);
    return SPAMM_OK;
}

// Per-row leaf task counts of A (x)_tau B over ALL rows (norms are replicated on
// every rank), for balancing a row partition on measured work.
extern "C" spamm_status spamm_row_task_counts(spamm_ctx ctx, spamm_mat A, spamm_mat B, double tau,
                                              int64_t *counts)
{
    if (!ctx || !A || !B || !counts) return set_err(ctx, SPAMM_EINVAL, "NULL argument");
    if (A->n != B->n || A->b != B->b) return set_err(ctx, SPAMM_ESHAPE, "shape mismatch");
    if (!(tau >= 0.0)) return set_err(ctx, SPAMM_EINVAL, "tau must be >= 0");
    Cull *cw = new Cull();
    cw->counts_only = true;
    spamm_status st = cull_run(ctx, cw, A, B, tau, 0, A->nb);
    if (ctx->last == cw) ctx->last = nullptr;
    std::vector<int32_t> code(cw->nsegs), len(cw->nsegs);
    if (!st && cw->nsegs) {
        cudaMemcpyAsync(code.data(), cw->seg_code, sizeof(int32_t) * cw->nsegs, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(len.data(), cw->seg_len, sizeof(int32_t) * cw->nsegs, cudaMemcpyDeviceToHost, ctx->stream);
        cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) st = check_cuda(ctx, e, "row task counts");
    }
    if (!st) {
        for (int i = 0; i < A->nb; i++) counts[i] = 0;
        for (int64_t t = 0; t < cw->nsegs; t++) counts[morton_i((uint32_t)code[t])] += len[t];
    }
    cull_free(ctx, cw);
    dev_free(ctx, cw->counters, sizeof(int32_t) * 64);
    if (cw->hcnt) cudaFreeHost(cw->hcnt);
    delete cw;
    return st;
}

// ------------------------------------------------ lensing instrumentation (f4)
// Histogram of the diagonal-plane distance d = max(|i-j|, |i-k|, |j-k|) of the
// last product's surviving leaf triples (the product-volume "lensing" of P:804-823,
// S:484): integer atomics, so the counts are exact and deterministic.
__global__ void k_task_dist_hist(const int4 *rec, int64_t n, int nbins, unsigned long long *hist)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int4 r = rec[t];
        const int i = morton_i((uint32_t)r.x), j = morton_j((uint32_t)r.x), k = r.y;
        int d = abs(i - j);
        d = max(d, abs(i - k));
        d = max(d, abs(j - k));
        atomicAdd(&hist[d < nbins ? d : nbins - 1], 1ull);
    }
}

static spamm_status task_hist(spamm_ctx ctx, Cull *cw, int64_t *hist, int32_t nbins)
{
    for (int b = 0; b < nbins; b++) hist[b] = 0;
    if (!cw || cw->ntasks == 0) return SPAMM_OK;
    unsigned long long *d = dalloc<unsigned long long>(ctx, nbins);
    if (!d) return set_err(ctx, SPAMM_ENOMEM, "histogram");
    CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * nbins, ctx->stream));
    const int grid = (int)std::min<int64_t>(cdiv(cw->ntasks, 256), 8 * ctx->sm_count);
    k_task_dist_hist<<<grid, 256, 0, ctx->stream>>>(cw->rec[cw->final_buf], cw->ntasks, nbins, d);
    CKL(ctx);
    CK(cudaMemcpyAsync(hist, d, sizeof(int64_t) * nbins, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    dev_free(ctx, d, sizeof(unsigned long long) * nbins);
    return SPAMM_OK;
}

extern "C" spamm_status spamm_task_distance_hist(spamm_ctx ctx, int64_t *hist, int32_t nbins)
{
    if (!ctx || !hist || nbins < 1) return set_err(ctx, SPAMM_EINVAL, "bad argument");
    return task_hist(ctx, ctx->last, hist, nbins);
}

extern "C" spamm_status spamm_ctx_set_volume_sink(spamm_ctx ctx, spamm_volume_sink *sink)
{
    if (!ctx) return SPAMM_EINVAL;
    if (sink && sink->nprod_cap < 0) return set_err(ctx, SPAMM_EINVAL, "nprod_cap < 0");
    ctx->vsink = sink;
    return SPAMM_OK;
}

spamm_status volume_record(spamm_ctx ctx, Cull *cw)
{
    spamm_volume_sink *v = ctx->vsink;
    if (!v) return SPAMM_OK;
    const int64_t p = v->nprod++;
    v->ikj_needed += cw->ntasks;
    if (p >= v->nprod_cap) return SPAMM_OK;
    if (v->ntasks) v->ntasks[p] = cw->ntasks;
    if (v->nbins > 0 && v->hist) ST(task_hist(ctx, cw, v->hist + p * v->nbins, v->nbins));
    if (v->ikj && v->ikj_count < v->ikj_cap) {
        int64_t n = 0;
        ST(cull_export(ctx, cw, v->ikj + 3 * v->ikj_count, v->ikj_cap - v->ikj_count, &n));
        v->ikj_count += std::min(n, v->ikj_cap - v->ikj_count);
    }
    return SPAMM_OK;
}
