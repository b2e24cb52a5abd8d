// comm.cu — transports of the row-partitioned path.
//
//   NcclComm  : one rank of an NCCL communicator (NVLink / NVSwitch between
//               B200s).  allgather = ncclAllGather; alltoallv = grouped
//               ncclSend / ncclRecv (the self part is a device copy).  NCCL is
//               resolved with dlopen so the library has no link-time NCCL
//               dependency (PyTorch's libnccl.so.2 is normally already loaded).
//   LocalComm : `world` ranks inside one process, one host thread and one
//               context (stream) per rank, on one device or several (peer access
//               enabled on first use).  Also offers peer memory (v3 of §8(e)):
//               ranks share device pointers and the GEMM reads remote tiles in place.
//               A collective is: publish buffers + a "ready" event, host
//               barrier, each rank pushes its data with stream-ordered copies
//               after waiting on the receivers' ready events, records "done",
//               barrier, waits on every sender's "done".  No kernel waits on
//               another rank's kernel; the copies are ordinary stream work.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "common.cuh"

// ------------------------------------------------------------------ NCCL
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
std::mutex g_nccl_mu;
NcclApi g_nccl;

template <typename F>
static bool sym(void *h, const char *name, F &f)
{
    f = reinterpret_cast<F>(dlsym(h, name));
    return f != nullptr;
}

NcclApi *nccl_api()
{
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) return g_nccl.ok ? &g_nccl : nullptr;
    g_nccl.tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    const char *env = getenv("SPAMM_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char *e = dlerror();
        g_nccl.why = e ? e : "dlopen(libnccl.so.2) failed";
        return nullptr;
    }
    NcclApi &a = g_nccl;
    bool ok = sym(h, "ncclGetUniqueId", a.GetUniqueId) && sym(h, "ncclCommInitRank", a.CommInitRank) &&
              sym(h, "ncclCommDestroy", a.CommDestroy) && sym(h, "ncclAllGather", a.AllGather) &&
              sym(h, "ncclSend", a.Send) && sym(h, "ncclRecv", a.Recv) &&
              sym(h, "ncclGroupStart", a.GroupStart) && sym(h, "ncclGroupEnd", a.GroupEnd) &&
              sym(h, "ncclGetErrorString", a.GetErrorString);
    sym(h, "ncclCommInitRankConfig", a.CommInitRankConfig);   // optional
    if (!ok) {
        a.why = "libnccl.so.2 lacks a required symbol";
        return nullptr;
    }
    a.ok = true;
    return &a;
}

struct NcclComm : spamm_comm_s {
    ncclComm_t comm = nullptr;
    NcclApi *api = nullptr;
    const char *kind() const override { return "nccl"; }
    ~NcclComm() override
    {
        if (comm && api) api->CommDestroy(comm);
    }
    spamm_status fail(spamm_ctx ctx, ncclResult_t r, const char *what)
    {
        return set_err(ctx, SPAMM_ENCCL, "NCCL %s failed: %s", what, api->GetErrorString(r));
    }
    spamm_status allgather(spamm_ctx ctx, const void *send, void *recv, size_t bytes) override
    {
        if (bytes == 0) return SPAMM_OK;
        ncclResult_t r = api->AllGather(send, recv, bytes, ncclUint8, comm, ctx->stream);
        return r == ncclSuccess ? SPAMM_OK : fail(ctx, r, "AllGather");
    }
    spamm_status alltoallv(spamm_ctx ctx, const void *send, const size_t *soff, const size_t *scnt, void *recv,
                           const size_t *roff, const size_t *rcnt) override
    {
        const char *s = (const char *)send;
        char *d = (char *)recv;
        if (scnt[rank] != rcnt[rank]) return set_err(ctx, SPAMM_EINVAL, "alltoallv: self counts differ");
        if (scnt[rank])
            CK(cudaMemcpyAsync(d + roff[rank], s + soff[rank], scnt[rank], cudaMemcpyDeviceToDevice, ctx->stream));
        ncclResult_t r = api->GroupStart();
        if (r != ncclSuccess) return fail(ctx, r, "GroupStart");
        for (int p = 0; p < world; p++) {
            if (p == rank) continue;
            if (scnt[p] && (r = api->Send(s + soff[p], scnt[p], ncclUint8, p, comm, ctx->stream)) != ncclSuccess)
                break;
            if (rcnt[p] && (r = api->Recv(d + roff[p], rcnt[p], ncclUint8, p, comm, ctx->stream)) != ncclSuccess)
                break;
        }
        ncclResult_t r2 = api->GroupEnd();
        if (r != ncclSuccess) return fail(ctx, r, "Send/Recv");
        return r2 == ncclSuccess ? SPAMM_OK : fail(ctx, r2, "GroupEnd");
    }
};

// ------------------------------------------------------------ local group
struct LocalShared {
    int world = 1;
    int refs = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    struct Slot {
        const void *send = nullptr;
        void *recv = nullptr;
        size_t bytes = 0;
        const size_t *soff = nullptr, *scnt = nullptr, *roff = nullptr, *rcnt = nullptr;
        cudaEvent_t ready = nullptr, done = nullptr;
        const void *const *ptrs = nullptr;   // peer_share: the published pointers
        int device = -1;
    };
    std::vector<Slot> slot;
    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        int64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LocalComm : spamm_comm_s {
    LocalShared *sh = nullptr;
    const char *kind() const override { return "local"; }
    ~LocalComm() override
    {
        LocalShared::Slot &me = sh->slot[rank];
        if (me.ready) cudaEventDestroy(me.ready);
        if (me.done) cudaEventDestroy(me.done);
        bool last;
        {
            std::lock_guard<std::mutex> lk(sh->mu);
            last = --sh->refs == 0;
        }
        if (last) delete sh;
    }
    spamm_status ensure_events(spamm_ctx ctx)
    {
        LocalShared::Slot &me = sh->slot[rank];
        if (!me.ready) CK(cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming));
        if (!me.done) CK(cudaEventCreateWithFlags(&me.done, cudaEventDisableTiming));
        return SPAMM_OK;
    }
    // phase 1: publish + ready; phase 2: push; phase 3: wait for every sender
    template <typename Push>
    spamm_status run(spamm_ctx ctx, Push push)
    {
        ST(ensure_events(ctx));
        LocalShared::Slot &me = sh->slot[rank];
        cudaError_t e1 = cudaEventRecord(me.ready, ctx->stream);
        sh->barrier();
        cudaError_t e2 = cudaSuccess;
        for (int p = 0; p < world && e2 == cudaSuccess; p++) {
            e2 = cudaStreamWaitEvent(ctx->stream, sh->slot[p].ready, 0);
            if (e2 == cudaSuccess) e2 = push(p);
        }
        if (e2 == cudaSuccess) e2 = cudaEventRecord(me.done, ctx->stream);
        sh->barrier();
        cudaError_t e3 = cudaSuccess;
        for (int p = 0; p < world && e3 == cudaSuccess; p++) e3 = cudaStreamWaitEvent(ctx->stream, sh->slot[p].done, 0);
        sh->barrier();  // slots may be reused by the next collective only now
        if (e1 != cudaSuccess) return check_cuda(ctx, e1, "local comm ready");
        if (e2 != cudaSuccess) return check_cuda(ctx, e2, "local comm push");
        if (e3 != cudaSuccess) return check_cuda(ctx, e3, "local comm wait");
        return SPAMM_OK;
    }
    bool peer_capable() const override { return true; }
    // publish + ready, barrier, read the peers' slots and wait for their ready events,
    // barrier (the slots may be reused by the next call only now)
    spamm_status peer_share(spamm_ctx ctx, const void *const *mine, int n, const void **all, int *ok) override
    {
        ST(ensure_events(ctx));
        LocalShared::Slot &me = sh->slot[rank];
        me.ptrs = mine;
        me.device = ctx->device;
        cudaError_t e1 = cudaEventRecord(me.ready, ctx->stream);
        sh->barrier();
        int can = 1;
        cudaError_t e2 = cudaSuccess;
        for (int p = 0; p < world && e2 == cudaSuccess; p++) {
            const LocalShared::Slot &q = sh->slot[p];
            for (int i = 0; i < n; i++) all[(size_t)p * n + i] = q.ptrs[i];
            if (q.device != ctx->device) {
                int a = 0;
                if (cudaDeviceCanAccessPeer(&a, ctx->device, q.device) != cudaSuccess || !a) can = 0;
                else if (cudaDeviceEnablePeerAccess(q.device, 0) == cudaErrorPeerAccessAlreadyEnabled)
                    cudaGetLastError();
            }
            e2 = cudaStreamWaitEvent(ctx->stream, q.ready, 0);
        }
        sh->barrier();
        *ok = can;
        if (e1 != cudaSuccess) return check_cuda(ctx, e1, "peer share ready");
        if (e2 != cudaSuccess) return check_cuda(ctx, e2, "peer share wait");
        return SPAMM_OK;
    }
    spamm_status peer_barrier(spamm_ctx ctx) override
    {
        ST(ensure_events(ctx));
        LocalShared::Slot &me = sh->slot[rank];
        cudaError_t e1 = cudaEventRecord(me.ready, ctx->stream);
        sh->barrier();
        cudaError_t e2 = cudaSuccess;
        for (int p = 0; p < world && e2 == cudaSuccess; p++) e2 = cudaStreamWaitEvent(ctx->stream, sh->slot[p].ready, 0);
        sh->barrier();
        if (e1 != cudaSuccess) return check_cuda(ctx, e1, "peer barrier ready");
        if (e2 != cudaSuccess) return check_cuda(ctx, e2, "peer barrier wait");
        return SPAMM_OK;
    }
    spamm_status allgather(spamm_ctx ctx, const void *send, void *recv, size_t bytes) override
    {
        LocalShared::Slot &me = sh->slot[rank];
        me.send = send;
        me.recv = recv;
        me.bytes = bytes;
        return run(ctx, [&](int p) -> cudaError_t {
            if (!bytes) return cudaSuccess;
            return cudaMemcpyAsync((char *)sh->slot[p].recv + (size_t)rank * bytes, send, bytes, cudaMemcpyDefault,
                                   ctx->stream);
        });
    }
    spamm_status alltoallv(spamm_ctx ctx, const void *send, const size_t *soff, const size_t *scnt, void *recv,
                           const size_t *roff, const size_t *rcnt) override
    {
        LocalShared::Slot &me = sh->slot[rank];
        me.send = send;
        me.recv = recv;
        me.soff = soff;
        me.scnt = scnt;
        me.roff = roff;
        me.rcnt = rcnt;
        return run(ctx, [&](int p) -> cudaError_t {
            // push my part for p into p's receive buffer at p's offset for me
            const LocalShared::Slot &dst = sh->slot[p];
            if (scnt[p] != dst.rcnt[rank]) return cudaErrorInvalidValue;
            if (!scnt[p]) return cudaSuccess;
            return cudaMemcpyAsync((char *)dst.recv + dst.roff[rank], (const char *)send + soff[p], scnt[p],
                                   cudaMemcpyDefault, ctx->stream);
        });
    }
};
}  // namespace

// ------------------------------------------------------------------ ABI
extern "C" spamm_status spamm_comm_nccl_unique_id(void *id128)
{
    if (!id128) return SPAMM_EINVAL;
    NcclApi *api = nccl_api();
    if (!api) return SPAMM_ENCCL;
    ncclUniqueId id;
    if (api->GetUniqueId(&id) != ncclSuccess) return SPAMM_ENCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(id128, &id, sizeof id);
    return SPAMM_OK;
}

extern "C" spamm_status spamm_comm_nccl_create(const void *id128, int32_t rank, int32_t world, int32_t device,
                                               spamm_comm *out)
{
    if (!id128 || !out || world < 1 || world > SPAMM_MAX_WORLD || rank < 0 || rank >= world) return SPAMM_EINVAL;
    *out = nullptr;
    NcclApi *api = nccl_api();
    if (!api) return SPAMM_ENCCL;
    if (cudaSetDevice(device) != cudaSuccess) return SPAMM_ECUDA;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    NcclComm *c = new NcclComm();
    c->api = api;
    c->rank = rank;
    c->world = world;
    // The halo exchange runs while the local-segment GEMM holds the SMs (spamm.cu
    // overlapped_gemm leaves exchange_ctas() SMs free): cap NCCL's CTAs to that many so
    // its kernels fit the reserved SMs instead of waiting for the GEMM to drain.
    ncclResult_t ir;
    if (api->CommInitRankConfig) {
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.maxCTAs = exchange_ctas();
        cfg.minCTAs = 1;
        ir = api->CommInitRankConfig(&c->comm, world, id, rank, &cfg);
    } else {
        ir = api->CommInitRank(&c->comm, world, id, rank);
    }
    if (ir != ncclSuccess) {
        c->comm = nullptr;
        delete c;
        return SPAMM_ENCCL;
    }
    *out = c;
    return SPAMM_OK;
}

extern "C" spamm_status spamm_comm_local_group(int32_t world, spamm_comm *comms)
{
    if (!comms || world < 1 || world > SPAMM_MAX_WORLD) return SPAMM_EINVAL;
    LocalShared *sh = new LocalShared();
    sh->world = world;
    sh->refs = world;
    sh->slot.resize(world);
    for (int r = 0; r < world; r++) {
        LocalComm *c = new LocalComm();
        c->sh = sh;
        c->rank = r;
        c->world = world;
        comms[r] = c;
    }
    return SPAMM_OK;
}

extern "C" void spamm_comm_destroy(spamm_comm comm) { delete comm; }
