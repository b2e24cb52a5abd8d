"""Row-partitioned path on one B200, through the C ABI.

G ranks run as host threads, each with its own library context and stream on
cuda:0, joined by the in-process communicator (spamm_comm_local_group: device
copies + host barriers, no kernel waits on another rank).  The claim under test
(DESIGN.md §7): every output block is computed by one rank with the same tasks
in the same k-order and the threshold comes from bitwise-replicated pyramids,
so products, t_k and the final Y, Z are BITWISE equal to the single-device
path for every world size and partition.  The single-device path is itself
pinned to the oracle in test_gpu_parity.py; one case here also checks the
assembled result against the oracle directly.  The NCCL transport runs at
world size 1 (one GPU per gpurun box).
"""
import numpy as np
import pytest

import oracle as O
import spamm_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def sp():
    import paper_1508_05856_b200 as m
    return m


def dist():
    from paper_1508_05856_b200 import dist as d
    return d


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return 0


@pytest.fixture(params=["peer", "halo"])
def transport(request, monkeypatch):
    """The in-process group's two transports: peer memory (v3, the default: the GEMM
    reads remote tiles in place from the owners' pools) and the halo exchange (v2,
    SPAMM_PEER=0, also what NCCL ranks use).  The library reads SPAMM_PEER per product."""
    monkeypatch.setenv("SPAMM_PEER", "1" if request.param == "peer" else "0")
    return {"peer": 2, "halo": 1}[request.param]


def gaussian(n, b, seed=150805856, sigma=0.8, tau_min=1e-7):
    cfg = si.Config("t", "gauss", n, b, 1e-7, 30, sigma=sigma, shift=1e-3, seed=seed, tau_min=tau_min)
    return si.make_input(cfg)[1]


def build(ctx, n, b, payload):
    if isinstance(payload, np.ndarray):
        return sp().spamm_build_tree(ctx, payload, b)
    bi, bj, blocks = payload
    return sp().spamm_build_tree_blocks(ctx, n, b, bi, bj, blocks)


def blocks_of(ctx, M):
    bi, bj, blk = sp().spamm_export_blocks(ctx, M)
    return {(int(i), int(j)): blk[t].copy() for t, (i, j) in enumerate(zip(bi, bj))}


def merged(results, key):
    out = {}
    for r in results:
        for k, v in r[key].items():
            assert k not in out, f"block {k} on two ranks"
            out[k] = v
    return out


def assert_bitwise(a: dict, b: dict):
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k


def single_ns(n, b, payload, tau, iters, mu=0.0):
    ctx = sp().spamm_ctx_create(0)
    S = build(ctx, n, b, payload)
    r = sp().spamm_ns_sqrt(ctx, S, tau, iters, mu=mu)
    out = dict(Y=blocks_of(ctx, r["Y"]), Z=blocks_of(ctx, r["Z"]), t=r["t"].copy(), c=r["c"],
               tasks=np.array([[p["tasks"] for p in k] for k in r["stats"]]),
               n2=sp().spamm_level_norms2(ctx, r["Y"], (n // b).bit_length() - 1))
    return out


def dist_ns(world, n, b, payload, tau, iters, row_start=None, mu=0.0, scale=0.0):
    def fn(rank, comm):
        ctx = sp().spamm_ctx_create(0, library_stream=True)
        sp().spamm_ctx_set_comm(ctx, comm, row_start)
        S = build(ctx, n, b, payload)
        r = sp().spamm_ns_sqrt(ctx, S, tau, iters, mu=mu, scale=scale)
        out = dict(Y=blocks_of(ctx, r["Y"]), Z=blocks_of(ctx, r["Z"]), t=r["t"].copy(), c=r["c"],
                   tasks=np.array([[p["tasks"] for p in k] for k in r["stats"]]),
                   transport={p["transport"] for k in r["stats"] for p in k},
                   rows=sp().spamm_mat_rows(r["Y"]),
                   n2=sp().spamm_level_norms2(ctx, r["Y"], (n // b).bit_length() - 1))
        for m in (S, r["Y"], r["Z"]):
            m.free()
        ctx.close()
        return out
    return dist().run_rank_threads(world, fn)


def check_same(ref, res, world, transport=None):
    if transport is not None and world > 1:
        assert all(r["transport"] == {transport} for r in res), [r["transport"] for r in res]
    assert_bitwise(merged(res, "Y"), ref["Y"])
    assert_bitwise(merged(res, "Z"), ref["Z"])
    for r in res:
        assert np.array_equal(r["t"].view(np.uint64), ref["t"].view(np.uint64))
        assert r["c"] == ref["c"]
        assert np.array_equal(r["n2"].view(np.uint64), ref["n2"].view(np.uint64))
    # every task is run by exactly one rank
    assert np.array_equal(sum(r["tasks"] for r in res), ref["tasks"])
    # the ranks' row ranges tile [0, nb) in rank order
    rows = [r["rows"] for r in res]
    assert rows[0][0] == 0 and all(rows[p][1] == rows[p + 1][0] for p in range(world - 1))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_ns_kms_bitwise_equal_to_single_device(gpu, world, transport):
    c = si.CONFIGS["C2"]
    s = si.kms(c.n, c.rho)
    iters = 12
    ref = single_ns(c.n, c.b, s, c.tau, iters)
    res = dist_ns(world, c.n, c.b, s, c.tau, iters)
    check_same(ref, res, world, transport)


@pytest.mark.parametrize("world,row_start", [(2, None), (4, None), (4, [0, 5, 6, 40, 64]),
                                             (8, None), (3, [0, 0, 64, 64])])
def test_ns_gaussian_bitwise(gpu, world, row_start, transport):
    """n = 4096, b = 64 (nb = 64) Gaussian overlap, uneven and empty ranges."""
    n, b = 4096, 64
    payload = gaussian(n, b)
    iters = 10
    ref = single_ns(n, b, payload, 1e-7, iters)
    res = dist_ns(world, n, b, payload, 1e-7, iters, row_start)
    check_same(ref, res, world, transport)
    if row_start is not None:
        assert [r["rows"] for r in res] == [(row_start[p], row_start[p + 1]) for p in range(world)]


def test_ns_dist_matches_oracle(gpu):
    """Assembled G=4 result vs the CPU oracle (free run, 1e-10)."""
    c = si.CONFIGS["C1"]
    s = si.kms(c.n, c.rho)
    So = O.OMat.from_dense(s, c.b)
    cs = O.power_scale(So)
    ro = O.ns_sqrt(So, c.tau, c.iters, scale=cs)
    res = dist_ns(4, c.n, c.b, s, c.tau, c.iters, scale=cs)
    Y = dist().assemble_dense(c.n, c.b, [(np.array([k[0] for k in r["Y"]]), np.array([k[1] for k in r["Y"]]),
                                          np.array(list(r["Y"].values()))) for r in res])
    Yo = ro["Y"].to_dense()
    assert np.linalg.norm(Y - Yo) / np.linalg.norm(Yo) <= 1e-10


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("tau", [0.0, 1e-6])
def test_multiply_bitwise_and_tasks(gpu, world, tau, transport):
    n, b = 2048, 32
    r = np.random.default_rng(7)
    i = np.arange(n)
    a = np.exp(-30.0 / n * np.abs(i[:, None] - i[None, :])) * r.standard_normal((n, n))
    a[:b, 2 * b:3 * b] = 0.0
    ctx = sp().spamm_ctx_create(0)
    A = build(ctx, n, b, a)
    C = sp().spamm_multiply(ctx, A, A, tau)
    ref = blocks_of(ctx, C)
    ref_tasks = {tuple(x) for x in sp().spamm_export_tasks(ctx)}
    counts = sp().spamm_row_task_counts(ctx, A, A, tau)
    assert counts.sum() == len(ref_tasks)

    def fn(rank, comm):
        c2 = sp().spamm_ctx_create(0, library_stream=True)
        sp().spamm_ctx_set_comm(c2, comm, dist().balanced_partition(counts, world))
        A2 = build(c2, n, b, a)
        C2, st = sp().spamm_multiply(c2, A2, A2, tau, want_stats=True)
        assert st["transport"] == transport
        out = (blocks_of(c2, C2), {tuple(x) for x in sp().spamm_export_tasks(c2)},
               sp().spamm_row_task_counts(c2, A2, A2, tau), sp().spamm_mat_rows(C2))
        A2.free()
        C2.free()
        c2.close()
        return out
    res = dist().run_rank_threads(world, fn)
    assert_bitwise(merged([{"C": x[0]} for x in res], "C"), ref)
    allt = set()
    for blocks, tasks, cnt, (r0, r1) in res:
        assert not (allt & tasks)
        allt |= tasks
        assert all(r0 <= t[0] < r1 for t in tasks)
        assert np.array_equal(cnt, counts)  # global counts from replicated norms
    assert allt == ref_tasks


def test_nccl_world1(gpu):
    """The NCCL transport (world size 1) runs the partitioned code path."""
    c = si.CONFIGS["C1"]
    s = si.kms(c.n, c.rho)
    ref = single_ns(c.n, c.b, s, c.tau, c.iters)
    uid = sp().spamm_comm_nccl_unique_id()
    comm = sp().spamm_comm_nccl_create(uid, 0, 1, 0)
    ctx = sp().spamm_ctx_create(0)
    sp().spamm_ctx_set_comm(ctx, comm)
    S = build(ctx, c.n, c.b, s)
    r = sp().spamm_ns_sqrt(ctx, S, c.tau, c.iters)
    assert_bitwise(blocks_of(ctx, r["Y"]), ref["Y"])
    assert_bitwise(blocks_of(ctx, r["Z"]), ref["Z"])
    for m in (S, r["Y"], r["Z"]):
        m.free()
    ctx.close()
    comm.destroy()


def test_partition_errors(gpu):
    comms = sp().spamm_comm_local_group(2)
    ctx = sp().spamm_ctx_create(0, library_stream=True)
    with pytest.raises(sp().SpammError):
        sp().spamm_ctx_set_comm(ctx, comms[0], [0, 9, 4])     # not ascending
    sp().spamm_ctx_set_comm(ctx, comms[0], [0, 4, 8])
    with pytest.raises(sp().SpammError) as e:                   # partition is for nb = 8
        build(ctx, 256, 16, si.kms(256, 0.5))
    assert e.value.code == 1
    sp().spamm_ctx_set_comm(ctx, None)
    ctx.close()
    for c in comms:
        c.destroy()


def test_ns_scaled_dist_bitwise(gpu):
    """The scaled map's second pass and the device-side alpha(t_k), eps(t_k) are
    replicated identically on every rank."""
    n, b = 4096, 64
    payload = gaussian(n, b)

    def run(ctx):
        S = build(ctx, n, b, payload)
        r = sp().spamm_ns_sqrt(ctx, S, 1e-7, 12, tau_s=1e-9, scaled=True)
        out = dict(Y=blocks_of(ctx, r["Y"]), Z=blocks_of(ctx, r["Z"]), t=r["t"].copy())
        for m in (S, r["Y"], r["Z"]):
            m.free()
        return out
    ref = run(sp().spamm_ctx_create(0))

    def fn(rank, comm):
        ctx = sp().spamm_ctx_create(0, library_stream=True)
        sp().spamm_ctx_set_comm(ctx, comm)
        out = run(ctx)
        ctx.close()
        return out
    res = dist().run_rank_threads(3, fn)
    assert_bitwise(merged(res, "Y"), ref["Y"])
    assert_bitwise(merged(res, "Z"), ref["Z"])
    for r in res:
        assert np.array_equal(r["t"].view(np.uint64), ref["t"].view(np.uint64))
