"""Host logic of the row-partitioned path on CPU (no GPU): partitions, and the
torch.distributed plumbing (gloo, world size 2) that bench.py and the NCCL
bootstrap use — unique-id broadcast, max / sum over ranks, gathering the
rank-local blocks of a result."""
import itertools
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1508_05856_b200 import dist as D


def test_equal_partition_matches_library_rule():
    for nb, w in [(64, 1), (64, 3), (256, 8), (5, 8), (2048, 7)]:
        rs = D.equal_partition(nb, w)
        assert rs[0] == 0 and rs[-1] == nb and len(rs) == w + 1
        assert all(rs[p] == (p * nb) // w for p in range(w + 1))
        assert all(rs[p] <= rs[p + 1] for p in range(w))


def brute_best(c, w):
    nb = len(c)
    best = None
    for cuts in itertools.combinations_with_replacement(range(nb + 1), w - 1):
        rs = [0, *cuts, nb]
        m = max(D.partition_loads(c, rs))
        best = m if best is None else min(best, m)
    return best


@pytest.mark.parametrize("seed", range(12))
def test_balanced_partition_optimal(seed):
    r = np.random.default_rng(seed)
    nb = int(r.integers(1, 9))
    w = int(r.integers(1, 5))
    c = r.integers(0, 50, nb)
    if seed % 3 == 0:
        c[r.integers(0, nb)] = 0
    rs = D.balanced_partition(c, w)
    assert len(rs) == w + 1 and rs[0] == 0 and rs[-1] == nb
    assert all(rs[p] <= rs[p + 1] for p in range(w))
    assert max(D.partition_loads(c, rs)) == brute_best(c, w)


def test_balanced_partition_skewed():
    c = np.zeros(100, dtype=np.int64)
    c[:10] = 1000        # dense head (e.g. boundary rows)
    c[10:] = 10
    rs = D.balanced_partition(c, 4)
    loads = D.partition_loads(c, rs)
    assert max(loads) <= 3000 and sum(loads) == c.sum()
    # deterministic
    assert rs == D.balanced_partition(c.copy(), 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # unique id: rank 0 draws (the library's ncclGetUniqueId needs no GPU), all ranks agree
        import paper_1508_05856_b200 as sp
        try:
            draw = sp.spamm_comm_nccl_unique_id
            draw()
        except Exception:  # noqa: BLE001 — NCCL not loadable here: any 128 bytes test the plumbing
            draw = lambda: bytes(np.random.default_rng(9).integers(0, 256, 128, dtype=np.uint8))  # noqa: E731
        uid = D.broadcast_unique_id(draw)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        out["ids_equal"] = all(x == ids[0] for x in ids) and len(uid) == 128
        # timing reductions used by bench.py
        out["max"] = D.max_over_ranks(1.5 + rank)
        out["sum"] = D.sum_over_ranks(10.0 * (rank + 1))
        # rank-local blocks of a row-partitioned result, gathered and assembled on rank 0
        n, b = 8, 2
        rs = D.equal_partition(n // b, world)
        bi = np.arange(rs[rank], rs[rank + 1], dtype=np.int32)
        blocks = np.stack([np.full((b, b), float(i)) for i in bi]) if len(bi) else np.zeros((0, b, b))
        parts = D.gather_to_rank0((bi, bi.copy(), blocks))
        if rank == 0:
            dense = D.assemble_dense(n, b, parts)
            out["dense_ok"] = bool(np.array_equal(np.diag(dense), np.repeat(np.arange(n // b), b).astype(float)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_plumbing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["ids_equal"]
        assert res[r]["max"] == 2.5
        assert res[r]["sum"] == 30.0
    assert res[0]["dense_ok"]


def test_assemble_rejects_duplicate_owner():
    blk = np.ones((1, 2, 2))
    with pytest.raises(ValueError):
        D.assemble_dense(4, 2, [(np.array([0]), np.array([0]), blk), (np.array([0]), np.array([0]), blk)])
