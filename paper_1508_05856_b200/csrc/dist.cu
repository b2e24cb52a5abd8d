// dist.cu — the row-partitioned SpAMM path (BASELINE.json
// north_star: "output block-rows are partitioned over GPUs; each step NCCL over
// NVLink all-gathers the operand blocks and norms each shard needs").
//
// Eq. newspamm gives C_ij = sum_k A_ik B_kj over the surviving k;
// output block row i needs A's row i (local: left operands are always
// row-partitioned like the output) and the B blocks (k, j) of its surviving
// tasks, where k runs over all rows.  The cull itself needs only norms, which
// are replicated.  So one product on rank g is:
//   1. cull restricted to output rows [r0, r1) (cull.cu, same kernels);
//   2. halo_exchange: mark the remote (k, j) blocks the local tasks use, compact
//      them in row-major (k, j) order — rows are contiguous per owner, so the
//      list comes out grouped by owner — exchange request counts (all-gather)
//      and request lists (send/recv), owners pack the requested blocks, blocks
//      come back by grouped send/recv into a halo pool, and the tasks' B slots
//      are patched to -(h+1) (the GEMM producer reads the halo for negatives);
//   3. the leaf GEMM on the local segments (unchanged);
//   4. norms_finish: all-gather the new leaf norms of the local rows, then the
//      pyramid is summed on every rank in the fixed single-device order.
// Every output block is computed by one rank with the same tasks in the same
// k-order, and T = tau^2 ||A||^2 ||B||^2 comes from bitwise-replicated
// pyramids, so results are bitwise independent of the world size.
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "scan.cuh"

spamm_status mat_parts(spamm_ctx ctx, int nb, Parts *p)
{
    memset(p, 0, sizeof *p);
    if (!ctx->comm) {
        p->world = 1;
        p->rs[0] = 0;
        p->rs[1] = nb;
        return SPAMM_OK;
    }
    const int W = ctx->comm->world;
    p->world = W;
    if (!ctx->row_start.empty()) {
        if ((int)ctx->row_start.size() != W + 1 || ctx->row_start[W] != nb)
            return set_err(ctx, SPAMM_EINVAL, "row partition is for nb=%d, matrix has nb=%d",
                           ctx->row_start.back(), nb);
        for (int q = 0; q <= W; q++) p->rs[q] = ctx->row_start[q];
    } else {
        for (int q = 0; q <= W; q++) p->rs[q] = (int)((int64_t)q * nb / W);
    }
    return SPAMM_OK;
}

static int max_rows(const Parts &p)
{
    int m = 0;
    for (int q = 0; q < p.world; q++) m = std::max(m, p.rs[q + 1] - p.rs[q]);
    return m;
}

// ----------------------------------------------------------- norm gather
__global__ void k_pack_leaf(const double *leaf, int nb, int r0, int r1, double *out)
{
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)(r1 - r0) * nb) return;
    int i = r0 + (int)(e / nb), j = (int)(e % nb);
    out[e] = leaf[morton(i, j)];
}

__global__ void k_unpack_leaf(const double *recv, int nb, Parts p, int maxrows, int self, double *leaf)
{
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)nb * nb) return;
    int i = (int)(e / nb), j = (int)(e % nb);
    int q = 0;
    while (q + 1 < p.world && p.rs[q + 1] <= i) q++;
    if (q == self) return;
    leaf[morton(i, j)] = recv[((int64_t)q * maxrows + (i - p.rs[q])) * nb + j];
}

spamm_status norms_finish(spamm_ctx ctx, spamm_mat m)
{
    if (m->dist && m->parts.world > 1) {
        const int nb = m->nb, mr = max_rows(m->parts), W = m->parts.world;
        const int64_t chunk = (int64_t)mr * nb;
        double *send = dalloc<double>(ctx, chunk), *recv = dalloc<double>(ctx, chunk * W);
        if (!send || !recv) return set_err(ctx, SPAMM_ENOMEM, "norm gather");
        double *leaf = m->norm2 + pyr_off(m->L);
        int64_t loc = (int64_t)(m->r1 - m->r0) * nb;
        if (loc > 0) {
            k_pack_leaf<<<cdiv(loc, 256), 256, 0, ctx->stream>>>(leaf, nb, m->r0, m->r1, send);
            CKL(ctx);
        }
        spamm_status st = ctx->comm->allgather(ctx, send, recv, sizeof(double) * chunk);
        if (!st) {
            k_unpack_leaf<<<cdiv((int64_t)nb * nb, 256), 256, 0, ctx->stream>>>(recv, nb, m->parts, mr,
                                                                               ctx->comm->rank, leaf);
            ctx->launches++;
        }
        dev_free(ctx, send, sizeof(double) * chunk);
        dev_free(ctx, recv, sizeof(double) * chunk * W);
        if (st) return st;
    }
    return pyramid_build(ctx, m);
}

spamm_status gather_rows(spamm_ctx ctx, const Parts &p, double *vec, int width)
{
    if (!ctx->comm || p.world <= 1) return SPAMM_OK;
    const int W = p.world, me = ctx->comm->rank, mr = max_rows(p);
    const int64_t chunk = (int64_t)mr * width;
    double *send = dalloc<double>(ctx, chunk), *recv = dalloc<double>(ctx, chunk * W);
    if (!send || !recv) return set_err(ctx, SPAMM_ENOMEM, "row gather");
    const int64_t loc = (int64_t)(p.rs[me + 1] - p.rs[me]) * width;
    if (loc) CK(cudaMemcpyAsync(send, vec + (int64_t)p.rs[me] * width, sizeof(double) * loc,
                                cudaMemcpyDeviceToDevice, ctx->stream));
    spamm_status st = ctx->comm->allgather(ctx, send, recv, sizeof(double) * chunk);
    for (int q = 0; q < W && !st; q++) {
        const int64_t cnt = (int64_t)(p.rs[q + 1] - p.rs[q]) * width;
        if (q == me || !cnt) continue;
        CK(cudaMemcpyAsync(vec + (int64_t)p.rs[q] * width, recv + q * chunk, sizeof(double) * cnt,
                           cudaMemcpyDeviceToDevice, ctx->stream));
    }
    dev_free(ctx, send, sizeof(double) * chunk);
    dev_free(ctx, recv, sizeof(double) * chunk * W);
    return st;
}

// ----------------------------------------------------------- halo exchange
// need[k*nb + j] = 1 for every remote (k, j) a local task uses (tB < 0).
__global__ void k_need_mark(const int4 *rec, int64_t n, const int32_t *tB, int nb, int32_t *need)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        if (tB[t] >= 0) continue;
        int4 r = rec[t];
        need[(int64_t)r.y * nb + morton_j((uint32_t)r.x)] = 1;
    }
}

// excl[x] = number of needed entries before x (row-major order); codes[excl[x]] = x.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_need_scan(const int32_t *need, int64_t count, ScanTiles<V1> st,
                                                       int32_t *excl)
{
    __shared__ V1 sw[THREADS / 32];
    __shared__ int s_tile, s_excl;
    int tile;
    while ((tile = next_tile(st.ticket, count, THREADS, &s_tile)) >= 0) {
        int64_t t = (int64_t)tile * THREADS + threadIdx.x;
        V1 v{(t < count && need[t]) ? 1 : 0};
        V1 tot;
        V1 ex = block_excl_scan<V1, THREADS>(v, &tot, sw);
        if (threadIdx.x < 32) {
            int e = tile_lookback(st, tile, tot).x;
            if (threadIdx.x == 0) s_excl = e;
        }
        __syncthreads();
        if (t < count) excl[t] = s_excl + ex.x;
        if (t == count - 1) excl[count] = s_excl + ex.x + v.x;
        __syncthreads();
    }
}

__global__ void k_owner_bounds(const int32_t *excl, int nb, Parts p, int64_t *bounds)
{
    int q = threadIdx.x;
    if (q <= p.world) bounds[q] = excl[(int64_t)p.rs[q] * nb];
}

__global__ void k_req_list(const int32_t *need, const int32_t *excl, int64_t count, int32_t *codes)
{
    int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x < count && need[x]) codes[excl[x]] = (int32_t)x;
}

// owner side: copy the requested blocks (pool layout, swizzle kept) into a send buffer
__global__ void k_pack_blocks(const int32_t *codes, int nb, const int32_t *slot, const double *pool, int b,
                              double *out)
{
    const int64_t t = blockIdx.x;
    const int x = codes[t];
    const int s = slot[morton(x / nb, x % nb)];
    const int64_t b2 = (int64_t)b * b;
    const double2 *src = reinterpret_cast<const double2 *>(pool + (int64_t)(s < 0 ? 0 : s) * b2);
    double2 *dst = reinterpret_cast<double2 *>(out + t * b2);
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    // a request for an absent block is an internal inconsistency: poison it (NaN)
    // so it surfaces as SPAMM_ENOTFINITE instead of a silently wrong product
    for (int e = threadIdx.x; e < b2 / 2; e += blockDim.x) dst[e] = s < 0 ? make_double2(nan, nan) : src[e];
}

__global__ void k_patch_tb(const int4 *rec, int64_t n, const int32_t *excl, int nb, int32_t *tB)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        if (tB[t] >= 0) continue;
        int4 r = rec[t];
        tB[t] = -(excl[(int64_t)r.y * nb + morton_j((uint32_t)r.x)] + 1);
    }
}

spamm_status halo_exchange(spamm_ctx ctx, Cull *cw, spamm_mat B, double **halo, int64_t *nhalo)
{
    *halo = nullptr;
    *nhalo = 0;
    if (!B->dist || B->parts.world <= 1) return SPAMM_OK;
    spamm_comm comm = ctx->comm;
    const Parts &P = B->parts;
    const int W = P.world, me = comm->rank, nb = B->nb, b = B->b;
    const int64_t N = (int64_t)nb * nb, b2 = (int64_t)b * b;
    const int64_t ntasks = cw->ntasks;
    const int4 *rec = cw->rec[cw->final_buf];
    cudaStream_t s = ctx->stream;

    int32_t *need = dalloc<int32_t>(ctx, N), *excl = dalloc<int32_t>(ctx, N + 1);
    const int ntiles = cdiv(N, 512);
    int32_t *flags = dalloc<int32_t>(ctx, ntiles + 1);
    V1 *agg = dalloc<V1>(ctx, ntiles), *pre = dalloc<V1>(ctx, ntiles);
    int64_t *dbounds = dalloc<int64_t>(ctx, W + 1 + W + W * W);
    int64_t *dmine = dbounds ? dbounds + W + 1 : nullptr, *dall = dmine ? dmine + W : nullptr;
    std::vector<int64_t> hb(W + 1), M((size_t)W * W);
    std::vector<size_t> soff(W), scnt(W), roff(W), rcnt(W);
    int32_t *codes = nullptr, *rcodes = nullptr;
    double *sendblk = nullptr, *hp = nullptr;
    int64_t total = 0, serve = 0;
    spamm_status st = SPAMM_OK;
    auto cleanup = [&]() {
        dev_free(ctx, need, sizeof(int32_t) * N);
        dev_free(ctx, excl, sizeof(int32_t) * (N + 1));
        dev_free(ctx, flags, sizeof(int32_t) * (ntiles + 1));
        dev_free(ctx, agg, sizeof(V1) * ntiles);
        dev_free(ctx, pre, sizeof(V1) * ntiles);
        dev_free(ctx, dbounds, sizeof(int64_t) * (W + 1 + W + W * W));
        dev_free(ctx, codes, sizeof(int32_t) * total);
        dev_free(ctx, rcodes, sizeof(int32_t) * serve);
        dev_free(ctx, sendblk, sizeof(double) * serve * b2);
    };
    // every exit (errors included) reaches cleanup()
    st = [&]() -> spamm_status {
        if (!need || !excl || !flags || !agg || !pre || !dbounds) return set_err(ctx, SPAMM_ENOMEM, "halo workspace");
        // 1. requests: mark, scan, per-owner bounds
        CK(cudaMemsetAsync(need, 0, sizeof(int32_t) * N, s));
        CK(cudaMemsetAsync(flags, 0, sizeof(int32_t) * (ntiles + 1), s));
        const int grid = (int)std::min<int64_t>(cdiv(std::max<int64_t>(ntasks, 1), 256), 8 * ctx->sm_count);
        k_need_mark<<<grid, 256, 0, s>>>(rec, ntasks, cw->tB, nb, need);
        CKL(ctx);
        ScanTiles<V1> tiles{flags, agg, pre, flags + ntiles};
        k_need_scan<512><<<std::min(ntiles, 2 * ctx->sm_count), 512, 0, s>>>(need, N, tiles, excl);
        CKL(ctx);
        k_owner_bounds<<<1, 96, 0, s>>>(excl, nb, P, dbounds);
        CKL(ctx);
        ST(fetch1(ctx, dbounds, hb.data(), sizeof(int64_t) * (W + 1)));
        total = hb[W];
        // 2. request counts: M[q][p] = blocks rank q wants from rank p
        std::vector<int64_t> mine(W);
        for (int p = 0; p < W; p++) mine[p] = hb[p + 1] - hb[p];
        CK(cudaMemcpyAsync(dmine, mine.data(), sizeof(int64_t) * W, cudaMemcpyHostToDevice, s));
        if ((st = comm->allgather(ctx, dmine, dall, sizeof(int64_t) * W))) return st;
        ST(fetch1(ctx, dall, M.data(), sizeof(int64_t) * W * W));
        for (int q = 0; q < W; q++) serve += M[(size_t)q * W + me];
        // 3. request lists to the owners
        codes = dalloc<int32_t>(ctx, total);
        rcodes = dalloc<int32_t>(ctx, serve);
        if (!codes || !rcodes) {
            st = set_err(ctx, SPAMM_ENOMEM, "halo request lists");
            return st;
        }
        k_req_list<<<cdiv(N, 256), 256, 0, s>>>(need, excl, N, codes);
        CKL(ctx);
        int64_t acc = 0;
        for (int p = 0; p < W; p++) {
            soff[p] = sizeof(int32_t) * hb[p];
            scnt[p] = sizeof(int32_t) * mine[p];
            rcnt[p] = sizeof(int32_t) * M[(size_t)p * W + me];
            roff[p] = sizeof(int32_t) * acc;
            acc += M[(size_t)p * W + me];
        }
        if ((st = comm->alltoallv(ctx, codes, soff.data(), scnt.data(), rcodes, roff.data(), rcnt.data()))) return st;
        // 4. owners pack, blocks come back into the halo in request order
        sendblk = dalloc<double>(ctx, serve * b2);
        hp = dalloc<double>(ctx, total * b2);
        if (!sendblk || !hp) {
            st = set_err(ctx, SPAMM_ENOMEM, "halo pool (%lld blocks)", (long long)total);
            return st;
        }
        if (serve) {
            k_pack_blocks<<<(int)serve, 256, 0, s>>>(rcodes, nb, B->slot, B->pool, b, sendblk);
            CKL(ctx);
        }
        acc = 0;
        for (int p = 0; p < W; p++) {
            const int64_t sv = M[(size_t)p * W + me];
            soff[p] = sizeof(double) * b2 * acc;
            scnt[p] = sizeof(double) * b2 * sv;
            acc += sv;
            roff[p] = sizeof(double) * b2 * hb[p];
            rcnt[p] = sizeof(double) * b2 * mine[p];
        }
        if ((st = comm->alltoallv(ctx, sendblk, soff.data(), scnt.data(), hp, roff.data(), rcnt.data()))) return st;
        // 5. tasks read remote tiles from the halo
        if (ntasks) {
            k_patch_tb<<<grid, 256, 0, s>>>(rec, ntasks, excl, nb, cw->tB);
            CKL(ctx);
        }
        return SPAMM_OK;
    }();
    cleanup();
    if (st) {
        dev_free(ctx, hp, sizeof(double) * total * b2);
        return st;
    }
    *halo = hp;
    *nhalo = total;
    return SPAMM_OK;
}

// ------------------------------------------------------------ peer memory
// §8(e) v3: where the ranks can read each other's memory (LocalComm: one process, one
// device or peer access over NVLink), the request / pack / send-recv sequence and the
// halo pool disappear.  The owners publish their pool and slot map; each remote task's
// B slot is resolved in the owner's slot map (a peer read) and encoded as
// tB = -(slot * W + owner) - 1; the GEMM producer bulk-copies those tiles straight from
// the owner's pool, so the transfer is overlapped with the DMMAs tile by tile by the
// GEMM's own pipeline.  Same tasks, same k order: bitwise the v2 and single-device
// results.
struct PeerSlots {
    const int32_t *p[SPAMM_MAX_WORLD];
};

__global__ void k_patch_tb_peer(const int4 *rec, int64_t n, int nb, Parts p, PeerSlots slots, int32_t *tB)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        if (tB[t] >= 0) continue;
        const int4 r = rec[t];
        const int k = r.y, j = morton_j((uint32_t)r.x);
        int q = 0;
        while (q + 1 < p.world && p.rs[q + 1] <= k) q++;
        const int s = slots.p[q][morton(k, j)];
        SPAMM_ASSERT(s >= 0);   // a surviving triple's B block is stored by its owner
        tB[t] = -(s * p.world + q) - 1;
    }
}

// SPAMM_PEER=0: the v2 halo exchange even where peer memory is available (read per
// product, so a test can switch it between runs)
static int peer_mode()
{
    const char *e = getenv("SPAMM_PEER");
    return e && *e ? atoi(e) : 1;
}

spamm_status peer_patch(spamm_ctx ctx, Cull *cw, spamm_mat B, bool *used)
{
    *used = false;
    cw->peer_world = 0;
    if (!B->dist || B->parts.world <= 1 || !ctx->comm || !ctx->comm->peer_capable() || !peer_mode())
        return SPAMM_OK;
    const int W = B->parts.world;
    const void *mine[2] = {B->pool, B->slot};
    std::vector<const void *> all((size_t)2 * W);
    int ok = 0;
    ST(ctx->comm->peer_share(ctx, mine, 2, all.data(), &ok));
    if (!ok) return SPAMM_OK;   // some pair cannot reach each other's memory: the v2 exchange
    PeerSlots ps{};
    for (int q = 0; q < W; q++) {
        cw->peer_pool[q] = static_cast<const double *>(all[(size_t)2 * q]);
        ps.p[q] = static_cast<const int32_t *>(all[(size_t)2 * q + 1]);
    }
    if (cw->ntasks > 0) {
        const int grid = (int)std::min<int64_t>(cdiv(cw->ntasks, 256), 8 * ctx->sm_count);
        k_patch_tb_peer<<<grid, 256, 0, ctx->stream>>>(cw->rec[cw->final_buf], cw->ntasks, B->nb, B->parts, ps, cw->tB);
        ctx->launches++;
        CKL(ctx);
    }
    cw->peer_world = W;
    *used = true;
    return SPAMM_OK;
}

// ------------------------------------------------- local-first segment order
// flag[s] = 1 iff every task of segment s reads a row-local B block (tB >= 0); those
// segments can run while the halo is in flight (overlap at
// segment granularity, never splitting a segment, so the k order is unchanged).
__global__ void k_seg_local(const int32_t *seg_start, const int32_t *seg_len, const int32_t *tB, int64_t nseg,
                            int32_t *flag)
{
    int64_t s = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= nseg) return;
    const int st = seg_start[s], len = seg_len[s];
    bool remote = false;
    for (int t = lane; t < len; t += 32) remote |= tB[st + t] < 0;
    remote = __any_sync(0xffffffffu, remote);
    if (lane == 0) flag[s] = remote ? 0 : 1;
}

// stable partition: local segments first (ascending), then the others (ascending)
__global__ void k_seg_order(const int32_t *flag, const int32_t *excl, int64_t nseg, int32_t *order)
{
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const int64_t nloc = excl[nseg];
    const int64_t pos = flag[s] ? excl[s] : nloc + (s - excl[s]);
    order[pos] = (int32_t)s;
}

spamm_status seg_split(spamm_ctx ctx, Cull *cw, int32_t **order, int64_t *nlocal)
{
    const int64_t ns = cw->nsegs;
    *order = nullptr;
    *nlocal = 0;
    cudaStream_t s = ctx->stream;
    int32_t *flag = dalloc<int32_t>(ctx, ns), *excl = dalloc<int32_t>(ctx, ns + 1);
    int32_t *ord = dalloc<int32_t>(ctx, ns);
    const int ntiles = cdiv(std::max<int64_t>(ns, 1), 512);
    int32_t *flags = dalloc<int32_t>(ctx, ntiles + 1);
    V1 *agg = dalloc<V1>(ctx, ntiles), *pre = dalloc<V1>(ctx, ntiles);
    spamm_status st = SPAMM_OK;
    int32_t h = 0;
    if (!flag || !excl || !ord || !flags || !agg || !pre) st = set_err(ctx, SPAMM_ENOMEM, "segment split");
    else if (ns > 0) {
        k_seg_local<<<cdiv(ns, 8), 256, 0, s>>>(cw->seg_start, cw->seg_len, cw->tB, ns, flag);
        ctx->launches++;
        cudaMemsetAsync(flags, 0, sizeof(int32_t) * (ntiles + 1), s);
        ScanTiles<V1> tiles{flags, agg, pre, flags + ntiles};
        k_need_scan<512><<<std::min(ntiles, 2 * ctx->sm_count), 512, 0, s>>>(flag, ns, tiles, excl);
        k_seg_order<<<cdiv(ns, 256), 256, 0, s>>>(flag, excl, ns, ord);
        ctx->launches += 2;
        st = fetch1(ctx, excl + ns, &h, sizeof(int32_t));
    }
    dev_free(ctx, flag, sizeof(int32_t) * ns);
    dev_free(ctx, excl, sizeof(int32_t) * (ns + 1));
    dev_free(ctx, flags, sizeof(int32_t) * (ntiles + 1));
    dev_free(ctx, agg, sizeof(V1) * ntiles);
    dev_free(ctx, pre, sizeof(V1) * ntiles);
    if (st) {
        dev_free(ctx, ord, sizeof(int32_t) * ns);
        return st;
    }
    *order = ord;
    *nlocal = h;
    return SPAMM_OK;
}

void dist_free(spamm_ctx ctx)
{
    if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    ctx->comm_stream = nullptr;
}

// ------------------------------------------------------------------ ABI
extern "C" spamm_status spamm_ctx_set_comm(spamm_ctx ctx, spamm_comm comm, const int32_t *row_start)
{
    if (!ctx) return SPAMM_EINVAL;
    ctx->row_start.clear();
    if (!comm) {
        ctx->comm = nullptr;
        return SPAMM_OK;
    }
    if (comm->world < 1 || comm->world > SPAMM_MAX_WORLD) return set_err(ctx, SPAMM_EINVAL, "bad world size");
    if (row_start) {
        if (row_start[0] != 0) return set_err(ctx, SPAMM_EINVAL, "row_start[0] must be 0");
        for (int q = 0; q < comm->world; q++)
            if (row_start[q + 1] < row_start[q]) return set_err(ctx, SPAMM_EINVAL, "row_start not ascending");
        ctx->row_start.assign(row_start, row_start + comm->world + 1);
    }
    ctx->comm = comm;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_mat_rows(spamm_mat m, int32_t *r0, int32_t *r1)
{
    if (!m) return SPAMM_EINVAL;
    if (r0) *r0 = m->r0;
    if (r1) *r1 = m->r1;
    return SPAMM_OK;
}
