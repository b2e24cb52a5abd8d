"""CPU oracle of SpAMM (x)_tau and the dual Newton-Schulz iteration (ctypes wrapper).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs are the only callers.  It shares no
code with ``paper_1508_05856_b200`` (the CUDA path) and never imports it.

The arithmetic lives in ``oracle/spamm_oracle.c`` (plain C, fp64, no fp
contraction, OpenMP task parallel recursion); each function there cites the
PAPER.md passage it follows.  This file only marshals arguments.

Parity status: every entry point is pinned by
``tests/test_oracle_pins.py`` except the exact iterate values at tau > 0, which
no paper number fixes ("parity unpinned vs paper": the figures of PAPER.md are
missing); those are pinned only indirectly (error bounds, convergence,
task-set brute force).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spamm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O3", "-march=native", "-ffp-contract=off", "-fno-fast-math",
          "-fopenmp", "-fPIC", "-shared", "-std=gnu11"]


def build(force: bool = False) -> str:
    """Compile oracle/spamm_oracle.c -> oracle/liboracle.so with gcc."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
        P = C.POINTER
        sig = {
            "or_build": (vp, [vp, i32, i32]),
            "or_build_blocks": (vp, [i32, i32, i64, vp, vp, vp]),
            "or_free": (None, [vp]),
            "or_norm": (dbl, [vp]),
            "or_n": (i32, [vp]),
            "or_b": (i32, [vp]),
            "or_to_dense": (None, [vp, vp]),
            "or_level_norms": (None, [vp, i32, vp]),
            "or_get_block": (i32, [vp, i32, i32, vp]),
            "or_nblocks": (i64, [vp]),
            "or_block_coords": (i64, [vp, vp, vp, i64]),
            "or_multiply": (vp, [vp, vp, dbl, vp, i64, P(i64)]),
            "or_copy": (vp, [vp]),
            "or_transpose": (vp, [vp]),
            "or_regularized_factor": (i32, [vp, dbl, dbl, vp, i32, i32, dbl, dbl, i32, P(vp), P(dbl), vp]),
            "or_multiply_t": (vp, [vp, vp, dbl, vp, i64, P(i64)]),
            "or_ns_sqrt_single": (i32, [vp, dbl, dbl, i32, dbl, i32, dbl, i32, P(vp), P(vp), vp, vp,
                                        P(dbl), P(C.c_int)]),
            "or_identity": (vp, [i32, i32]),
            "or_scale": (vp, [vp, dbl, i32]),
            "or_trace": (dbl, [vp]),
            "or_power_scale": (dbl, [vp, i32]),
            "or_ns_step": (i32, [vp, vp, dbl, dbl, P(vp), P(vp), P(vp), P(dbl), vp]),
            "or_ns_y0": (vp, [vp, dbl, dbl]),
            "or_ns_sqrt": (i32, [vp, dbl, dbl, i32, dbl, i32, dbl, dbl, i32, P(vp), P(vp), vp, vp,
                                 P(dbl), P(C.c_int)]),
            "or_ns_step_map": (i32, [vp, vp, dbl, dbl, i32, P(vp), P(vp), P(vp), P(dbl), vp]),
            "or_ns_step_tasks": (i32, [vp, vp, dbl, dbl, i32, P(vp), P(vp), P(vp), P(dbl), vp, vp, vp, vp, i64]),
            "or_alpha": (dbl, [dbl]),
            "or_eps": (dbl, [dbl]),
            "or_num_threads": (i32, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OMat:
    """Owning handle of an oracle quadtree matrix."""

    def __init__(self, h):
        if not h:
            raise ValueError("oracle: invalid matrix (shape / tau precondition failed)")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_free(self.h)
            self.h = None

    # construction ---------------------------------------------------------
    @classmethod
    def from_dense(cls, s: np.ndarray, b: int) -> "OMat":
        s = np.ascontiguousarray(s, dtype=np.float64)
        assert s.ndim == 2 and s.shape[0] == s.shape[1]
        return cls(lib().or_build(_ptr(s), s.shape[0], b))

    @classmethod
    def from_blocks(cls, n: int, b: int, bi, bj, blocks) -> "OMat":
        bi = np.ascontiguousarray(bi, dtype=np.int32)
        bj = np.ascontiguousarray(bj, dtype=np.int32)
        blocks = np.ascontiguousarray(blocks, dtype=np.float64)
        return cls(lib().or_build_blocks(n, b, len(bi), _ptr(bi), _ptr(bj), _ptr(blocks)))

    @classmethod
    def identity(cls, n: int, b: int) -> "OMat":
        return cls(lib().or_identity(n, b))

    # queries --------------------------------------------------------------
    @property
    def n(self) -> int:
        return lib().or_n(self.h)

    @property
    def b(self) -> int:
        return lib().or_b(self.h)

    @property
    def nb(self) -> int:
        return self.n // self.b

    def norm(self) -> float:
        return lib().or_norm(self.h)

    def trace(self) -> float:
        return lib().or_trace(self.h)

    def to_dense(self) -> np.ndarray:
        out = np.empty((self.n, self.n))
        lib().or_to_dense(self.h, _ptr(out))
        return out

    def level_norms(self, level: int) -> np.ndarray:
        side = 1 << level
        out = np.empty((side, side))
        lib().or_level_norms(self.h, level, _ptr(out))
        return out

    def leaf_norms(self) -> np.ndarray:
        L = self.nb.bit_length() - 1
        return self.level_norms(L)

    def block(self, I: int, J: int):
        out = np.empty((self.b, self.b))
        present = lib().or_get_block(self.h, I, J, _ptr(out))
        return out if present else None

    def nblocks(self) -> int:
        return lib().or_nblocks(self.h)

    def block_coords(self):
        nbk = self.nblocks()
        bi = np.empty(nbk, dtype=np.int32)
        bj = np.empty(nbk, dtype=np.int32)
        lib().or_block_coords(self.h, _ptr(bi), _ptr(bj), nbk)
        return bi, bj

    def copy(self) -> "OMat":
        return OMat(lib().or_copy(self.h))


def multiply(A: OMat, B: OMat, tau: float, want_tasks: bool = False, trans_a: bool = False):
    """C = A (x)_tau B (Eq. newspamm), or A^T (x)_tau B with trans_a.  Returns C or
    (C, tasks[ntasks,3] = (i,k,j) sorted lexicographically)."""
    n = C.c_int64(0)
    fn = lib().or_multiply_t if trans_a else lib().or_multiply
    if not want_tasks:
        h = fn(A.h, B.h, float(tau), None, 0, C.byref(n))
        return OMat(h)
    cap = 1 << 16
    while True:
        buf = np.empty(3 * cap, dtype=np.int32)
        h = fn(A.h, B.h, float(tau), _ptr(buf), cap, C.byref(n))
        if n.value <= cap:
            t = buf[: 3 * n.value].reshape(-1, 3)
            t = t[np.lexsort((t[:, 1], t[:, 2], t[:, 0]))]   # sort by (i, j, k)
            return OMat(h), t
        lib().or_free(h)
        cap = int(n.value)


def power_scale(s: OMat, K: int = 100) -> float:
    return lib().or_power_scale(s.h, K)


def ns_y0(s: OMat, c: float, mu: float = 0.0) -> OMat:
    return OMat(lib().or_ns_y0(s.h, c, mu))


def _sort_tasks(t):
    return t[np.lexsort((t[:, 1], t[:, 2], t[:, 0]))]   # by (i, j, k)


def ns_step(Y: OMat, Z: OMat, tau: float, tau_s: float | None = None, scaled: bool = False,
            want_tasks: bool = False, task_cap: int = 1 << 16, allow_nonfinite: bool = False):
    """One dual NS step (north_star form). Returns (Y', Z', H, t, counts[3]), plus the
    three products' leaf triples [X, Y', Z'] (each [ntasks, 3] sorted by (i, j, k)) with
    want_tasks.  allow_nonfinite: return the non-finite iterates instead of raising."""
    tau_s = tau if tau_s is None else tau_s
    while True:
        yn, zn, hn = C.c_void_p(), C.c_void_p(), C.c_void_p()
        t = C.c_double(0)
        counts = np.zeros(3, dtype=np.int64)
        bufs = [np.empty(3 * task_cap, dtype=np.int32) for _ in range(3)] if want_tasks else None
        tp = [_ptr(x) for x in bufs] if want_tasks else [None, None, None]
        rc = lib().or_ns_step_tasks(Y.h, Z.h, tau, tau_s, int(scaled), C.byref(yn), C.byref(zn), C.byref(hn),
                                    C.byref(t), _ptr(counts), *tp, task_cap if want_tasks else 0)
        out = (OMat(yn.value), OMat(zn.value), OMat(hn.value), t.value, counts)
        if want_tasks and counts.max() > task_cap:
            task_cap = int(counts.max())
            continue
        break
    if rc and not allow_nonfinite:
        raise FloatingPointError("oracle NS step: non-finite iterate")
    if want_tasks:
        out = out + ([_sort_tasks(b[: 3 * c].reshape(-1, 3)) for b, c in zip(bufs, counts)],)
    return out


def ns_sqrt(s: OMat, tau: float, iters: int, tau_s: float | None = None,
            scale: float = 0.0, mu: float = 0.0, power_iters: int = 100, t_stop: float = 0.0,
            scaled: bool = False):
    """Full dual NS run. Returns dict(Y, Z, t, counts, c, rc, iters); t_stop > 0 stops
    after the first k with |t_k| <= t_stop (t, counts then cover the steps run)."""
    tau_s = tau if tau_s is None else tau_s
    yo, zo = C.c_void_p(), C.c_void_p()
    t = np.zeros(iters)
    counts = np.zeros(3 * iters, dtype=np.int64)
    c = C.c_double(0)
    done = C.c_int(0)
    rc = lib().or_ns_sqrt(s.h, tau, tau_s, iters, scale, power_iters, mu, t_stop, int(scaled), C.byref(yo),
                          C.byref(zo), _ptr(t), _ptr(counts), C.byref(c), C.byref(done))
    k = done.value if rc == 0 else done.value + 1   # keep the failing step's t_k
    return dict(Y=OMat(yo.value), Z=OMat(zo.value), t=t[:k], counts=counts.reshape(iters, 3)[:k],
                c=c.value, rc=rc, iters=k)


def num_threads() -> int:
    return lib().or_num_threads()


def alpha(t: float) -> float:
    """Scaling sigmoid alpha(t) of P:442-445."""
    return lib().or_alpha(float(t))


def eps(t: float) -> float:
    """Stabilisation sigmoid eps(t) of P:446-448."""
    return lib().or_eps(float(t))


def transpose(A: OMat) -> OMat:
    """A^T with the node norms carried over (||a^T|| = ||a||)."""
    return OMat(lib().or_transpose(A.h))


def ns_sqrt_single(s: OMat, tau: float, iters: int, tau_s: float | None = None, scale: float = 0.0,
                   power_iters: int = 100, t_stop: float = 0.0, scaled: bool = False):
    """Single-channel run: Z <- Z (x) h[X], W = s (x)_tau_s Z, X <- Z^T (x) W.
    Returns dict(Y = W sqrt(c), Z, t, counts[k] = (ZH, sZ, Z^T W), c, rc, iters)."""
    tau_s = tau if tau_s is None else tau_s
    yo, zo = C.c_void_p(), C.c_void_p()
    t = np.zeros(iters)
    counts = np.zeros(3 * iters, dtype=np.int64)
    c = C.c_double(0)
    done = C.c_int(0)
    rc = lib().or_ns_sqrt_single(s.h, tau, tau_s, iters, scale, power_iters, t_stop, int(scaled), C.byref(yo),
                                 C.byref(zo), _ptr(t), _ptr(counts), C.byref(c), C.byref(done))
    k = done.value if rc == 0 else done.value + 1
    return dict(Y=OMat(yo.value), Z=OMat(zo.value), t=t[:k], counts=counts.reshape(iters, 3)[:k],
                c=c.value, rc=rc, iters=k)


def regularized_factor(s: OMat, tau0: float, tau1: float, mus, iters: int, t_stop: float = 0.0,
                       scale: float = 0.0, power_iters: int = 100):
    """Regularised product representation: returns dict(G, c, slice_iters, rc) with
    G^T (s + c mu_m I) G ~ I."""
    mu = np.ascontiguousarray(mus, dtype=np.float64)
    g = C.c_void_p()
    c = C.c_double(0)
    its = np.zeros(len(mu), dtype=np.int64)
    rc = lib().or_regularized_factor(s.h, tau0, tau1, _ptr(mu), len(mu), iters, t_stop, scale, power_iters,
                                     C.byref(g), C.byref(c), _ptr(its))
    return dict(G=OMat(g.value), c=c.value, slice_iters=its, rc=rc)
