"""paper_1508_05856_b200 — B200 (sm_100a) SpAMM and dual Newton-Schulz.

Thin ctypes binding over the C ABI of ``libspamm_b200.so`` (``include/spamm.h``).
Function names are the C names; this module only marshals arguments (torch
tensors / numpy arrays -> raw pointers, handles -> objects).  Every step of
the method runs in the library's CUDA kernels.  PyTorch supplies device memory
(its caching allocator, passed to the library as allocator callbacks) and the
CUDA stream.  There is no CPU fallback: if the library cannot be loaded, or
there is no sm_100 device, the calls raise.

Method: Challacombe, Haut & Bock, arXiv 1508.05856 — SpAMM (Eq. newspamm,
PAPER.md P:199-216) inside the dual-channel Newton-Schulz square-root
iteration (Eq. cannonical).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build

__all__ = [
    "SpammError", "Ctx", "Mat", "load",
    "spamm_ctx_create", "spamm_ctx_destroy", "spamm_last_error", "spamm_kernel_launches",
    "spamm_build_tree", "spamm_build_tree_blocks", "spamm_mat_free", "spamm_mat_info",
    "spamm_norm", "spamm_to_dense", "spamm_level_norms2", "spamm_get_blocks",
    "spamm_multiply", "spamm_multiply_t", "spamm_task_distance_hist", "spamm_regularized_factor", "spamm_ns_step_single", "spamm_ns_sqrt_single", "spamm_export_tasks", "spamm_ns_step", "spamm_ns_step_map", "spamm_power_scale",
    "spamm_ns_y0", "spamm_identity", "spamm_ns_sqrt", "spamm_scale",
    "spamm_export_blocks", "spamm_profile_enable", "spamm_profile_read", "spamm_peak_dmma",
    "Comm", "spamm_comm_nccl_unique_id", "spamm_comm_nccl_create", "spamm_comm_local_group",
    "spamm_comm_destroy", "spamm_ctx_set_comm", "spamm_mat_rows", "spamm_row_task_counts",
    "VolumeSink", "spamm_ctx_set_volume_sink",
    "spamm_export_blocks_async", "spamm_copies_join", "spamm_copies_wait",
    "spamm_stage_blocks", "spamm_stage_dense", "spamm_build_tree_staged", "spamm_staged_free",
]

STATUS = {0: "SPAMM_OK", 1: "SPAMM_EINVAL", 2: "SPAMM_ESHAPE", 3: "SPAMM_ENOMEM",
          4: "SPAMM_ECUDA", 5: "SPAMM_ENCCL", 6: "SPAMM_ENOTFINITE", 7: "SPAMM_ECAPACITY"}


class SpammError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class spamm_stats(C.Structure):
    _fields_ = [("tasks", C.c_int64), ("segments", C.c_int64), ("candidates", C.c_int64),
                ("level_survivors", C.c_int64 * 24), ("flops", C.c_double), ("halo_blocks", C.c_int64),
                ("local_segments", C.c_int64), ("transport", C.c_int32)]

    def as_dict(self):
        return dict(tasks=self.tasks, segments=self.segments, candidates=self.candidates,
                    level_survivors=list(self.level_survivors), flops=self.flops,
                    halo_blocks=self.halo_blocks, local_segments=self.local_segments,
                    transport=self.transport)


class spamm_ns_opts(C.Structure):
    _fields_ = [("tau_s", C.c_double), ("mu", C.c_double), ("scale", C.c_double),
                ("power_iters", C.c_int32), ("t_history", C.c_void_p),
                ("per_product", C.c_void_p), ("c_out", C.c_void_p), ("t_stop", C.c_double),
                ("iters_done", C.c_void_p), ("map", C.c_int32)]


NPHASE = 5
PHASES = ("gemm", "cull", "setup", "loop", "other")


class spamm_profile_t(C.Structure):
    _fields_ = [("ms", C.c_double * NPHASE), ("count", C.c_int64 * NPHASE),
                ("gemm_flops", C.c_double), ("gemm_tasks", C.c_int64),
                ("gemm_operand_bytes", C.c_double)]


class spamm_volume_sink(C.Structure):
    _fields_ = [("nbins", C.c_int32), ("hist", C.c_void_p), ("ntasks", C.c_void_p), ("ikj", C.c_void_p),
                ("ikj_cap", C.c_int64), ("nprod_cap", C.c_int64), ("nprod", C.c_int64),
                ("ikj_count", C.c_int64), ("ikj_needed", C.c_int64)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class spamm_allocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


_LIB = None


def load():
    """Load (building in-tree first if needed) libspamm_b200.so."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("SPAMM_LIB", _build.LIB)   # SPAMM_LIB: an experimental build (A/B timing)
    if not os.path.exists(path):
        path = _build.build()
    L = C.CDLL(path)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    sigs = {
        "spamm_ctx_create": (i32, [C.c_int, vp, P(spamm_allocator), P(vp)]),
        "spamm_ctx_destroy": (None, [vp]),
        "spamm_last_error": (C.c_char_p, [vp]),
        "spamm_kernel_launches": (i64, [vp]),
        "spamm_build_tree": (i32, [vp, vp, i64, i64, i32, P(vp)]),
        "spamm_build_tree_blocks": (i32, [vp, i64, i32, i64, vp, vp, vp, P(vp)]),
        "spamm_mat_free": (None, [vp]),
        "spamm_mat_info": (i32, [vp, P(i64), P(i32), P(i64)]),
        "spamm_norm": (i32, [vp, vp, P(dbl)]),
        "spamm_to_dense": (i32, [vp, vp, vp, i64]),
        "spamm_level_norms2": (i32, [vp, vp, i32, vp]),
        "spamm_get_blocks": (i32, [vp, vp, i64, vp, vp, vp, vp]),
        "spamm_multiply": (i32, [vp, vp, vp, dbl, P(vp), P(spamm_stats)]),
        "spamm_export_tasks": (i32, [vp, vp, i64, P(i64)]),
        "spamm_multiply_t": (i32, [vp, vp, vp, dbl, P(vp), P(spamm_stats)]),
        "spamm_task_distance_hist": (i32, [vp, vp, i32]),
        "spamm_regularized_factor": (i32, [vp, vp, dbl, dbl, vp, i32, i32, dbl, dbl, P(vp), P(dbl), vp]),
        "spamm_ns_step_single": (i32, [vp, vp, vp, vp, dbl, dbl, i32, P(vp), P(vp), P(vp), P(dbl), vp, vp]),
        "spamm_ns_sqrt_single": (i32, [vp, vp, dbl, i32, P(vp), P(vp), P(spamm_ns_opts)]),
        "spamm_ns_step": (i32, [vp, vp, vp, dbl, dbl, P(vp), P(vp), P(vp), P(dbl), vp]),
        "spamm_ns_step_map": (i32, [vp, vp, vp, dbl, dbl, i32, P(vp), P(vp), P(vp), P(dbl), vp, vp]),
        "spamm_power_scale": (i32, [vp, vp, i32, P(dbl)]),
        "spamm_ns_y0": (i32, [vp, vp, dbl, dbl, P(vp)]),
        "spamm_identity": (i32, [vp, i64, i32, P(vp)]),
        "spamm_ns_sqrt": (i32, [vp, vp, dbl, i32, P(vp), P(vp), P(spamm_ns_opts)]),
        "spamm_scale": (i32, [vp, vp, dbl, i32, P(vp)]),
        "spamm_export_blocks": (i32, [vp, vp, vp, vp, vp, i64, P(i64)]),
        "spamm_profile_enable": (i32, [vp, i32]),
        "spamm_profile_read": (i32, [vp, P(spamm_profile_t)]),
        "spamm_peak_dmma": (i32, [vp, i64, P(dbl), P(dbl)]),
        "spamm_comm_nccl_unique_id": (i32, [vp]),
        "spamm_comm_nccl_create": (i32, [vp, i32, i32, i32, P(vp)]),
        "spamm_comm_local_group": (i32, [i32, vp]),
        "spamm_comm_destroy": (None, [vp]),
        "spamm_ctx_set_comm": (i32, [vp, vp, vp]),
        "spamm_mat_rows": (i32, [vp, P(i32), P(i32)]),
        "spamm_row_task_counts": (i32, [vp, vp, vp, dbl, vp]),
        "spamm_ctx_set_volume_sink": (i32, [vp, vp]),
        "spamm_export_blocks_async": (i32, [vp, vp, vp, vp, vp, i64, P(i64)]),
        "spamm_copies_join": (i32, [vp]),
        "spamm_copies_wait": (i32, [vp]),
        "spamm_stage_blocks": (i32, [vp, i64, i32, vp, vp, vp, P(vp)]),
        "spamm_stage_dense": (i32, [vp, vp, i64, i64, P(vp)]),
        "spamm_build_tree_staged": (i32, [vp, i64, i32, vp, P(vp)]),
        "spamm_staged_free": (None, [vp]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def exported_symbols():
    """Names declared in include/spamm.h that the binding resolves."""
    load()
    return [n for n in __all__ if n.startswith("spamm_")]


# --------------------------------------------------------------- marshalling
def _ptr(x):
    """Raw pointer of a torch tensor (host or device) or numpy array."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return C.c_void_p(x.ctypes.data)
    assert x.is_contiguous()
    return C.c_void_p(x.data_ptr())


class Ctx:
    """A library context bound to a CUDA device and (torch's current) stream.

    library_stream=True gives the context its own stream and the library's
    cudaMallocAsync allocator (used when several host threads drive one device
    each with its own context, e.g. the in-process rank group)."""

    def __init__(self, device: int = 0, stream=None, torch_allocator: bool = True,
                 library_stream: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise SpammError(4, "no CUDA device: the SpAMM library has no CPU path")
        L = load()
        self.torch = torch
        self.device = device
        self.comm = None
        torch.cuda.set_device(device)
        if library_stream:
            stream, torch_allocator = None, False
        elif stream is None:
            stream = torch.cuda.current_stream(device)
            if stream.cuda_stream == 0:
                # the legacy default stream: give the library a real torch stream so
                # that events recorded on ctx.stream bracket the library's own work
                stream = torch.cuda.Stream(device)
        self.stream = stream
        self._keep = []
        alloc_p = None
        if torch_allocator:
            raw_alloc = torch._C._cuda_cudaCachingAllocator_raw_alloc
            raw_delete = torch._C._cuda_cudaCachingAllocator_raw_delete

            def _alloc(nbytes, strm, user):
                try:
                    return raw_alloc(int(nbytes), strm or 0)
                except Exception:  # noqa: BLE001 — reported as SPAMM_ENOMEM by the library
                    return None

            def _free(ptr, nbytes, strm, user):
                raw_delete(ptr)

            a = spamm_allocator(ALLOC_FN(_alloc), FREE_FN(_free), None)
            self._keep = [a, _alloc, _free]
            alloc_p = C.byref(a)
        h = C.c_void_p()
        rc = L.spamm_ctx_create(device, C.c_void_p(stream.cuda_stream if stream is not None else None),
                                alloc_p, C.byref(h))
        if rc:
            raise SpammError(rc, "spamm_ctx_create failed (device must be sm_100)")
        self.h = h

    def sync_in(self):
        """Order the library stream after torch's current stream (device inputs)."""
        if self.stream is not None:
            self.stream.wait_stream(self.torch.cuda.current_stream(self.device))

    def sync_out(self):
        """Order torch's current stream after the library stream (device outputs)."""
        if self.stream is not None:
            self.torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def check(self, rc):
        if rc:
            raise SpammError(rc, load().spamm_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            load().spamm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class Mat:
    """Owning handle of a device-resident quadtree matrix."""

    def __init__(self, ctx: Ctx, h):
        self.ctx = ctx
        self.h = h

    def free(self):
        # valid after ctx.close() too: the library defers a context's teardown to the
        # last spamm_mat_free of its matrices (the allocator callbacks stay alive with
        # self.ctx)
        if getattr(self, "h", None):
            load().spamm_mat_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass

    def info(self):
        n, b, nblk = C.c_int64(), C.c_int32(), C.c_int64()
        self.ctx.check(load().spamm_mat_info(self.h, C.byref(n), C.byref(b), C.byref(nblk)))
        return n.value, b.value, nblk.value

    @property
    def n(self):
        return self.info()[0]

    @property
    def b(self):
        return self.info()[1]

    @property
    def nblocks(self):
        return self.info()[2]


class Comm:
    """Owning handle of one rank of a communicator (NCCL or in-process group)."""

    def __init__(self, h, rank: int, world: int, kind: str):
        self.h, self.rank, self.world, self.kind = h, rank, world, kind

    def destroy(self):
        if getattr(self, "h", None):
            load().spamm_comm_destroy(self.h)
            self.h = None


# ------------------------------------------------------------------- calls
def spamm_ctx_create(device: int = 0, stream=None, torch_allocator: bool = True,
                     library_stream: bool = False) -> Ctx:
    return Ctx(device, stream, torch_allocator, library_stream)


def spamm_comm_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = load().spamm_comm_nccl_unique_id(buf)
    if rc:
        raise SpammError(rc, "ncclGetUniqueId failed (NCCL not loadable?)")
    return buf.raw


def spamm_comm_nccl_create(uid: bytes, rank: int, world: int, device: int) -> Comm:
    assert len(uid) == 128
    h = C.c_void_p()
    buf = C.create_string_buffer(uid, 128)
    rc = load().spamm_comm_nccl_create(buf, rank, world, device, C.byref(h))
    if rc:
        raise SpammError(rc, f"ncclCommInitRank failed (rank {rank} of {world})")
    return Comm(h, rank, world, "nccl")


def spamm_comm_local_group(world: int) -> list:
    hs = (C.c_void_p * world)()
    rc = load().spamm_comm_local_group(world, hs)
    if rc:
        raise SpammError(rc, "spamm_comm_local_group failed")
    return [Comm(C.c_void_p(hs[r]), r, world, "local") for r in range(world)]


def spamm_comm_destroy(comm: Comm):
    comm.destroy()


def spamm_ctx_set_comm(ctx: Ctx, comm: Comm | None, row_start=None):
    """Attach a communicator and the block-row partition (row_start[world+1], or
    None for the equal split) to ctx; matrices built afterwards are row-partitioned."""
    rs = None
    if row_start is not None:
        rs = np.ascontiguousarray(row_start, dtype=np.int32)
        assert comm is not None and rs.shape == (comm.world + 1,)
    ctx.check(load().spamm_ctx_set_comm(ctx.h, comm.h if comm is not None else None, _ptr(rs)))
    ctx.comm = comm


def spamm_mat_rows(m: Mat):
    r0, r1 = C.c_int32(), C.c_int32()
    m.ctx.check(load().spamm_mat_rows(m.h, C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def spamm_row_task_counts(ctx: Ctx, A: Mat, B: Mat, tau: float) -> np.ndarray:
    nb = A.n // A.b
    out = np.zeros(nb, dtype=np.int64)
    ctx.check(load().spamm_row_task_counts(ctx.h, A.h, B.h, float(tau), _ptr(out)))
    return out


def spamm_ctx_destroy(ctx: Ctx):
    ctx.close()


def spamm_last_error(ctx: Ctx) -> str:
    return load().spamm_last_error(ctx.h).decode()


def spamm_kernel_launches(ctx: Ctx) -> int:
    return load().spamm_kernel_launches(ctx.h)


def spamm_build_tree(ctx: Ctx, dense, b: int) -> Mat:
    """dense: n x n row-major fp64 torch tensor (cuda or cpu) or numpy array."""
    n = dense.shape[0]
    h = C.c_void_p()
    ctx.sync_in()
    ctx.check(load().spamm_build_tree(ctx.h, _ptr(dense), n, dense.shape[1], b, C.byref(h)))
    return Mat(ctx, h)


def spamm_build_tree_blocks(ctx: Ctx, n: int, b: int, bi, bj, blocks) -> Mat:
    h = C.c_void_p()
    ctx.sync_in()
    ctx.check(load().spamm_build_tree_blocks(ctx.h, n, b, len(bi), _ptr(bi), _ptr(bj),
                                             _ptr(blocks), C.byref(h)))
    return Mat(ctx, h)


def spamm_mat_free(m: Mat):
    m.free()


def spamm_mat_info(m: Mat):
    return m.info()


def spamm_norm(ctx: Ctx, m: Mat) -> float:
    v = C.c_double()
    ctx.check(load().spamm_norm(ctx.h, m.h, C.byref(v)))
    return v.value


def spamm_to_dense(ctx: Ctx, m: Mat, out=None, device: bool = True):
    """Dense copy as a torch tensor (device=True) or numpy array."""
    n = m.n
    if out is None:
        if device:
            out = ctx.torch.empty((n, n), dtype=ctx.torch.float64, device=f"cuda:{ctx.device}")
        else:
            out = np.empty((n, n))
    if not isinstance(out, np.ndarray):
        ctx.sync_in()          # the output buffer was allocated on torch's stream
    ctx.check(load().spamm_to_dense(ctx.h, m.h, _ptr(out), out.shape[1]))
    if not isinstance(out, np.ndarray):
        ctx.sync_out()
    return out


def spamm_level_norms2(ctx: Ctx, m: Mat, level: int) -> np.ndarray:
    side = 1 << level
    out = np.empty((side, side))
    ctx.check(load().spamm_level_norms2(ctx.h, m.h, level, _ptr(out)))
    return out


def spamm_get_blocks(ctx: Ctx, m: Mat, bi, bj):
    bi = np.ascontiguousarray(bi, dtype=np.int32)
    bj = np.ascontiguousarray(bj, dtype=np.int32)
    b = m.b
    out = np.empty((len(bi), b, b))
    pres = np.empty(len(bi), dtype=np.int32)
    ctx.check(load().spamm_get_blocks(ctx.h, m.h, len(bi), _ptr(bi), _ptr(bj), _ptr(out), _ptr(pres)))
    return out, pres.astype(bool)


def spamm_multiply(ctx: Ctx, A: Mat, B: Mat, tau: float, want_stats: bool = False):
    h = C.c_void_p()
    st = spamm_stats()
    ctx.check(load().spamm_multiply(ctx.h, A.h, B.h, float(tau), C.byref(h), C.byref(st)))
    m = Mat(ctx, h)
    return (m, st.as_dict()) if want_stats else m


def spamm_multiply_t(ctx: Ctx, A: Mat, B: Mat, tau: float, want_stats: bool = False):
    """C = A^T (x)_tau B."""
    h = C.c_void_p()
    st = spamm_stats()
    ctx.check(load().spamm_multiply_t(ctx.h, A.h, B.h, float(tau), C.byref(h), C.byref(st)))
    m = Mat(ctx, h)
    return (m, st.as_dict()) if want_stats else m


def spamm_ns_step_single(ctx: Ctx, S1: Mat, Z: Mat, H: Mat, tau: float, tau_s: float | None = None,
                         scaled: bool = False, want_w: bool = False):
    """One single-channel step; returns (Z', H', t', stats[3], (alpha, eps) [, W])."""
    tau_s = tau if tau_s is None else tau_s
    zn, hn, wn = C.c_void_p(), C.c_void_p(), C.c_void_p()
    t = C.c_double()
    ae = (C.c_double * 2)()
    sts = (spamm_stats * 3)()
    ctx.check(load().spamm_ns_step_single(ctx.h, S1.h, Z.h, H.h, float(tau), float(tau_s), int(scaled),
                                          C.byref(zn), C.byref(hn), C.byref(wn) if want_w else None,
                                          C.byref(t), sts, ae))
    out = (Mat(ctx, zn), Mat(ctx, hn), t.value, [s.as_dict() for s in sts], (ae[0], ae[1]))
    return out + (Mat(ctx, wn),) if want_w else out


def spamm_ns_sqrt_single(ctx: Ctx, s: Mat, tau: float, iters: int, tau_s: float | None = None,
                         scale: float = 0.0, power_iters: int = 100, t_stop: float = 0.0,
                         scaled: bool = False):
    """Full single-channel run: returns dict(Y, Z, t, stats, c, iters)."""
    t = np.zeros(iters)
    sts = (spamm_stats * (3 * iters))()
    c = C.c_double()
    done = C.c_int32(0)
    o = spamm_ns_opts(-1.0 if tau_s is None else float(tau_s), 0.0, float(scale), int(power_iters),
                      t.ctypes.data, C.cast(sts, C.c_void_p), C.cast(C.pointer(c), C.c_void_p), float(t_stop),
                      C.cast(C.pointer(done), C.c_void_p), int(scaled))
    yo, zo = C.c_void_p(), C.c_void_p()
    ctx.check(load().spamm_ns_sqrt_single(ctx.h, s.h, float(tau), int(iters), C.byref(yo), C.byref(zo),
                                          C.byref(o)))
    k = done.value
    stats = [[sts[3 * j + p].as_dict() for p in range(3)] for j in range(k)]
    return dict(Y=Mat(ctx, yo), Z=Mat(ctx, zo), t=t[:k], stats=stats, c=c.value, iters=k)


def spamm_task_distance_hist(ctx: Ctx, nbins: int) -> np.ndarray:
    """Histogram of max(|i-j|, |i-k|, |j-k|) over the last product's leaf triples."""
    out = np.zeros(nbins, dtype=np.int64)
    ctx.check(load().spamm_task_distance_hist(ctx.h, _ptr(out), int(nbins)))
    return out


def spamm_regularized_factor(ctx: Ctx, s: Mat, tau0: float, tau1: float, mus, iters: int,
                             t_stop: float = 0.0, scale: float = 0.0):
    """Regularised product representation: dict(G, c, slice_iters) with
    G^T (s + c mu_m I) G ~ I."""
    mu = np.ascontiguousarray(mus, dtype=np.float64)
    g = C.c_void_p()
    c = C.c_double()
    its = np.zeros(len(mu), dtype=np.int32)
    ctx.check(load().spamm_regularized_factor(ctx.h, s.h, float(tau0), float(tau1), _ptr(mu), len(mu), int(iters),
                                              float(t_stop), float(scale), C.byref(g), C.byref(c), _ptr(its)))
    return dict(G=Mat(ctx, g), c=c.value, slice_iters=its)


def spamm_export_tasks(ctx: Ctx) -> np.ndarray:
    """Leaf triples (i,k,j) of the last product: [ntasks, 3] int32."""
    n = C.c_int64()
    ctx.check(load().spamm_export_tasks(ctx.h, None, 0, C.byref(n)))
    buf = np.empty(3 * max(n.value, 1), dtype=np.int32)
    ctx.check(load().spamm_export_tasks(ctx.h, _ptr(buf), n.value, C.byref(n)))
    return buf[: 3 * n.value].reshape(-1, 3)


def spamm_ns_step(ctx: Ctx, Y: Mat, Z: Mat, tau: float, tau_s: float | None = None,
                  want_h: bool = False):
    """One dual NS step; returns (Y', Z', t_k, [stats X, Y', Z'] [, H])."""
    tau_s = tau if tau_s is None else tau_s
    yn, zn, hn = C.c_void_p(), C.c_void_p(), C.c_void_p()
    t = C.c_double()
    sts = (spamm_stats * 3)()
    ctx.check(load().spamm_ns_step(ctx.h, Y.h, Z.h, float(tau), float(tau_s), C.byref(yn),
                                   C.byref(zn), C.byref(hn) if want_h else None, C.byref(t), sts))
    out = (Mat(ctx, yn), Mat(ctx, zn), t.value, [s.as_dict() for s in sts])
    return out + (Mat(ctx, hn),) if want_h else out


def spamm_ns_step_map(ctx: Ctx, Y: Mat, Z: Mat, tau: float, tau_s: float | None = None,
                      scaled: bool = True, want_h: bool = False):
    """One dual NS step with the chosen map; returns (Y', Z', t_k, stats, (alpha, eps) [, H])."""
    tau_s = tau if tau_s is None else tau_s
    yn, zn, hn = C.c_void_p(), C.c_void_p(), C.c_void_p()
    t = C.c_double()
    ae = (C.c_double * 2)()
    sts = (spamm_stats * 3)()
    ctx.check(load().spamm_ns_step_map(ctx.h, Y.h, Z.h, float(tau), float(tau_s), int(scaled), C.byref(yn),
                                       C.byref(zn), C.byref(hn) if want_h else None, C.byref(t), sts, ae))
    out = (Mat(ctx, yn), Mat(ctx, zn), t.value, [s.as_dict() for s in sts], (ae[0], ae[1]))
    return out + (Mat(ctx, hn),) if want_h else out


def spamm_power_scale(ctx: Ctx, s: Mat, K: int = 100) -> float:
    c = C.c_double()
    ctx.check(load().spamm_power_scale(ctx.h, s.h, K, C.byref(c)))
    return c.value


def spamm_ns_y0(ctx: Ctx, s: Mat, c: float, mu: float = 0.0) -> Mat:
    h = C.c_void_p()
    ctx.check(load().spamm_ns_y0(ctx.h, s.h, float(c), float(mu), C.byref(h)))
    return Mat(ctx, h)


def spamm_identity(ctx: Ctx, n: int, b: int) -> Mat:
    h = C.c_void_p()
    ctx.check(load().spamm_identity(ctx.h, n, b, C.byref(h)))
    return Mat(ctx, h)


def spamm_scale(ctx: Ctx, m: Mat, alpha: float, divide: bool = False) -> Mat:
    h = C.c_void_p()
    ctx.check(load().spamm_scale(ctx.h, m.h, float(alpha), int(divide), C.byref(h)))
    return Mat(ctx, h)


def spamm_ns_sqrt(ctx: Ctx, s: Mat, tau: float, iters: int, tau_s: float | None = None,
                  mu: float = 0.0, scale: float = 0.0, power_iters: int = 100,
                  want_stats: bool = True, t_stop: float = 0.0, scaled: bool = False,
                  check: bool = True):
    """Full dual NS run: returns dict(Y, Z, t, stats, c, iters).  t_stop > 0 ends the
    run after the first k with |t_k| <= t_stop (t, stats then cover the steps run).
    check=False: a failing run returns dict(status=<code>, error=<text>, t=<history up to
    the failing step>, iters=<steps completed>) instead of raising."""
    t = np.zeros(iters)
    sts = (spamm_stats * (3 * iters))() if want_stats else None
    c = C.c_double()
    done = C.c_int32(0)
    o = spamm_ns_opts(-1.0 if tau_s is None else float(tau_s), float(mu), float(scale),
                      int(power_iters), t.ctypes.data, C.cast(sts, C.c_void_p) if want_stats else None,
                      C.cast(C.pointer(c), C.c_void_p), float(t_stop),
                      C.cast(C.pointer(done), C.c_void_p), int(scaled))
    yo, zo = C.c_void_p(), C.c_void_p()
    rc = load().spamm_ns_sqrt(ctx.h, s.h, float(tau), int(iters), C.byref(yo), C.byref(zo), C.byref(o))
    if rc and not check:
        k = done.value
        return dict(status=rc, error=load().spamm_last_error(ctx.h).decode(), t=t[:k + 1], iters=k, c=c.value)
    ctx.check(rc)
    k = done.value
    stats = None
    if want_stats:
        stats = [[sts[3 * j + p].as_dict() for p in range(3)] for j in range(k)]
    return dict(Y=Mat(ctx, yo), Z=Mat(ctx, zo), t=t[:k], stats=stats, c=c.value, iters=k)


def spamm_export_blocks(ctx: Ctx, m: Mat, out=None):
    """All stored blocks: (bi, bj, blocks).  out = (bi, bj, blocks) preallocated
    torch tensors (pinned host or device) or None for numpy."""
    n = C.c_int64()
    ctx.check(load().spamm_export_blocks(ctx.h, m.h, None, None, None, 0, C.byref(n)))
    k = n.value
    if out is None:
        b = m.b
        out = (np.empty(k, dtype=np.int32), np.empty(k, dtype=np.int32), np.empty((k, b, b)))
    bi, bj, blocks = out
    ctx.sync_in()
    ctx.check(load().spamm_export_blocks(ctx.h, m.h, _ptr(bi), _ptr(bj), _ptr(blocks), k,
                                         C.byref(n)))
    ctx.sync_out()
    return bi[:k], bj[:k], blocks[:k]


def spamm_export_blocks_async(ctx: Ctx, m: Mat, out):
    """Asynchronous export into preallocated HOST buffers out = (bi, bj, blocks) (pinned
    torch tensors or numpy arrays); valid after spamm_copies_wait / spamm_copies_join.
    Returns the number of blocks."""
    bi, bj, blocks = out
    n = C.c_int64()
    ctx.check(load().spamm_export_blocks_async(ctx.h, m.h, _ptr(bi), _ptr(bj), _ptr(blocks), len(bi),
                                               C.byref(n)))
    return n.value


class Staged:
    """Handle of an upload in flight (spamm_stage_blocks); keeps the host arrays alive."""

    def __init__(self, ctx, h, keep):
        self.ctx, self.h, self.keep = ctx, h, keep

    def __del__(self):
        if getattr(self, "h", None):
            load().spamm_staged_free(self.h)
            self.h = None


def spamm_stage_blocks(ctx: Ctx, b: int, bi, bj, blocks) -> Staged:
    """Start the upload of a HOST block list (pinned torch tensors or numpy arrays)."""
    h = C.c_void_p()
    ctx.check(load().spamm_stage_blocks(ctx.h, len(bi), b, _ptr(bi), _ptr(bj), _ptr(blocks), C.byref(h)))
    return Staged(ctx, h, (bi, bj, blocks))


def spamm_stage_dense(ctx: Ctx, dense) -> Staged:
    """Start the upload of a HOST dense n x n row-major matrix (pinned tensor / numpy)."""
    h = C.c_void_p()
    ctx.check(load().spamm_stage_dense(ctx.h, _ptr(dense), dense.shape[0], dense.shape[1], C.byref(h)))
    return Staged(ctx, h, (dense,))


def spamm_build_tree_staged(ctx: Ctx, n: int, b: int, staged: Staged) -> Mat:
    """Build from a staged upload (consumes the handle)."""
    h = C.c_void_p()
    sh, staged.h = staged.h, None
    ctx.check(load().spamm_build_tree_staged(ctx.h, n, b, sh, C.byref(h)))
    return Mat(ctx, h)


def spamm_copies_join(ctx: Ctx):
    ctx.check(load().spamm_copies_join(ctx.h))


def spamm_copies_wait(ctx: Ctx):
    ctx.check(load().spamm_copies_wait(ctx.h))


def spamm_profile_enable(ctx: Ctx, enable: bool = True):
    ctx.check(load().spamm_profile_enable(ctx.h, int(enable)))


def spamm_profile_read(ctx: Ctx) -> dict:
    p = spamm_profile_t()
    ctx.check(load().spamm_profile_read(ctx.h, C.byref(p)))
    d = {f"{ph}_ms": p.ms[i] for i, ph in enumerate(PHASES)}
    d.update({f"{ph}_count": p.count[i] for i, ph in enumerate(PHASES)})
    d.update(gemm_flops=p.gemm_flops, gemm_tasks=p.gemm_tasks,
             gemm_operand_bytes=p.gemm_operand_bytes)
    return d


def spamm_peak_dmma(ctx: Ctx, iters: int = 200000):
    t, ms = C.c_double(), C.c_double()
    ctx.check(load().spamm_peak_dmma(ctx.h, int(iters), C.byref(t), C.byref(ms)))
    return t.value, ms.value


class VolumeSink:
    """Host buffers of the per-product volume recorder (spamm_volume_sink, §8(f) f4).

    After the recorded calls: ``ntasks[p]``, ``hist[p]`` (distance histogram) and
    ``tasks(p)`` (the (i,k,j) triples of product p, if ikj_cap covered them)."""

    def __init__(self, nprod_cap: int, nbins: int = 0, ikj_cap: int = 0):
        self.hist_buf = np.zeros((nprod_cap, max(nbins, 1)), dtype=np.int64)
        self.ntasks_buf = np.zeros(nprod_cap, dtype=np.int64)
        self.ikj_buf = np.zeros((max(ikj_cap, 1), 3), dtype=np.int32)
        self.s = spamm_volume_sink(int(nbins), self.hist_buf.ctypes.data if nbins > 0 else None,
                                   self.ntasks_buf.ctypes.data, self.ikj_buf.ctypes.data if ikj_cap > 0 else None,
                                   int(ikj_cap), int(nprod_cap), 0, 0, 0)

    @property
    def nprod(self) -> int:
        return self.s.nprod

    @property
    def ntasks(self) -> np.ndarray:
        return self.ntasks_buf[: min(self.s.nprod, len(self.ntasks_buf))]

    @property
    def hist(self) -> np.ndarray:
        return self.hist_buf[: min(self.s.nprod, len(self.hist_buf))]

    def complete(self) -> bool:
        """True if every recorded triple fit in ikj_cap."""
        return self.s.ikj_count == self.s.ikj_needed

    def tasks(self, p: int) -> np.ndarray:
        off = int(self.ntasks_buf[:p].sum())
        n = int(self.ntasks_buf[p])
        assert off + n <= self.s.ikj_count, "ikj_cap too small for product %d" % p
        return self.ikj_buf[off: off + n]


def spamm_ctx_set_volume_sink(ctx: Ctx, sink: VolumeSink | None):
    """Attach (or detach with None) a per-product volume recorder to ctx."""
    ctx.check(load().spamm_ctx_set_volume_sink(ctx.h, C.byref(sink.s) if sink is not None else None))
    ctx._vsink = sink   # the library holds raw pointers into it


def spamm_staged_free(staged: Staged):
    """Drop an upload handle that will not be built."""
    if getattr(staged, "h", None):
        load().spamm_staged_free(staged.h)
        staged.h = None
