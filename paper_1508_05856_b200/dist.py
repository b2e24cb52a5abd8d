"""Host-side plumbing of the row-partitioned path.

Argument marshalling and orchestration only — no SpAMM arithmetic lives here:
  * row partitions of the nb leaf block rows (equal split, or balanced on
    measured per-row task counts from ``spamm_row_task_counts``);
  * NCCL communicator bootstrap: rank 0 draws the unique id through the C ABI
    and torch.distributed broadcasts it (gloo or nccl process group);
  * an in-process rank group (one host thread + one library context per rank)
    that runs G ranks on one device for the determinism tests;
  * max / sum over ranks of device timings (bench.py), and gathering the
    rank-local blocks of a result.
"""
from __future__ import annotations

import threading

import numpy as np


def equal_partition(nb: int, world: int) -> list[int]:
    """row_start[world+1] with rank p owning block rows [floor(p*nb/W), floor((p+1)*nb/W))
    (the library's default when no partition is given)."""
    return [(p * nb) // world for p in range(world + 1)]


def balanced_partition(costs, world: int) -> list[int]:
    """Contiguous block-row ranges minimising the largest per-rank cost.

    costs: per-row non-negative work (e.g. leaf task counts).  Binary search on
    the bottleneck value with a greedy feasibility check (exact for contiguous
    partitions of non-negative weights); ties resolved toward earlier cuts, so
    the result is deterministic.  Every rank gets a (possibly empty) range."""
    c = np.asarray(costs, dtype=np.int64)
    nb = c.shape[0]
    if world <= 1 or nb == 0:
        return [0] + [nb] * max(world, 1)

    def cuts_for(limit):
        cuts, acc = [0], 0
        for i in range(nb):
            if acc + c[i] > limit and acc > 0:
                cuts.append(i)
                acc = 0
            acc += c[i]
        return cuts

    lo, hi = int(c.max(initial=0)), int(c.sum())
    while lo < hi:
        mid = (lo + hi) // 2
        if len(cuts_for(mid)) <= world:
            hi = mid
        else:
            lo = mid + 1
    cuts = cuts_for(lo)
    # pad with empty trailing ranges
    while len(cuts) < world:
        cuts.append(nb)
    return cuts + [nb]


def partition_loads(costs, row_start) -> list[int]:
    c = np.asarray(costs, dtype=np.int64)
    return [int(c[row_start[p]:row_start[p + 1]].sum()) for p in range(len(row_start) - 1)]


# ------------------------------------------------------------------ NCCL
def broadcast_unique_id(draw, group=None) -> bytes:
    """Rank 0 calls draw() -> 128 bytes; every rank returns the same bytes
    (torch.distributed.broadcast_object_list over the default or given group)."""
    import torch.distributed as dist
    obj = [draw() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    return bytes(uid)


def init_nccl_comm(device: int, group=None):
    """One NCCL communicator over the torch.distributed world, created by the
    library (spamm_comm_nccl_create) from a broadcast unique id."""
    import torch.distributed as dist

    import paper_1508_05856_b200 as sp
    uid = broadcast_unique_id(sp.spamm_comm_nccl_unique_id, group)
    return sp.spamm_comm_nccl_create(uid, dist.get_rank(), dist.get_world_size(), device)


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def assemble_dense(n: int, b: int, parts) -> np.ndarray:
    """Dense n x n matrix from per-rank (bi, bj, blocks) lists.  Block rows are
    disjoint across ranks; a block reported twice is an error."""
    out = np.zeros((n, n))
    seen = set()
    for bi, bj, blocks in parts:
        for I, J, blk in zip(np.asarray(bi), np.asarray(bj), np.asarray(blocks)):
            key = (int(I), int(J))
            if key in seen:
                raise ValueError(f"block {key} owned by two ranks")
            seen.add(key)
            out[I * b:(I + 1) * b, J * b:(J + 1) * b] = blk
    return out


def gather_to_rank0(obj):
    """torch.distributed.gather_object to rank 0 (list on rank 0, None elsewhere)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [obj]
    out = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(obj, out, dst=0)
    return out


# ------------------------------------------------------- in-process group
def run_rank_threads(world: int, fn, timeout: float = 600.0):
    """Run fn(rank, comm) for rank = 0..world-1, each in its own host thread with
    one rank of an in-process communicator (spamm_comm_local_group).  Returns the
    per-rank results; re-raises the first exception."""
    import paper_1508_05856_b200 as sp
    comms = sp.spamm_comm_local_group(world)
    res = [None] * world
    err = [None] * world

    def body(r):
        try:
            res[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001 — re-raised in the caller
            err[r] = e

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
        if t.is_alive():
            raise TimeoutError("rank thread did not finish (a peer failed before a collective?)")
    for e in err:
        if e is not None:
            raise e
    for c in comms:
        c.destroy()
    return res
