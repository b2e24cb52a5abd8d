"""Parity at BASELINE.json's full sizes, in the configuration bench.py times (B200).

Lockstep: the GPU produces the input iterates (Y_k, Z_k) of a run (same tau,
tau_s, seeded input), they are exported, and the CPU oracle runs the same dual
step from them (Eq. cannonical in the north_star form, Eq. newspamm products).
Compared, SURVEY.md §8(c) / north_star (BJ:5):
  * the three products' task SETS (recorded per product by the volume sink):
    identical except triples within 1e-12 of the threshold;
  * t_k to 1e-12 (absolute, or relative once |t| > 1);
  * the block patterns of H, Y', Z' identical; the values over the union of both
    sides' blocks (C3: every block; C4/C5: a seeded sample of 1500 blocks drawn
    from the union), relative Frobenius <= 1e-12 after the flip correction.
Free run: C3 exactly as BASELINE.json configs[2] gives it (tau_s = tau, 30 fixed
iterations, c from the oracle), every block of Y and Z <= 1e-10, all 90 task
counts identical, t_k to 1e-12.
The oracle runs on the box's host cores (up to ~2e12 flop per C5 step).
"""
import math

import numpy as np
import pytest

import _parity as P
import oracle as O
import spamm_inputs as si

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def sp():
    import paper_1508_05856_b200 as m
    return m


def export(ctx, M, n, b):
    bi, bj, blk = sp().spamm_export_blocks(ctx, M)
    return O.OMat.from_blocks(n, b, bi, bj, blk)


def keys(tr, nb):
    t = np.asarray(tr, dtype=np.int64).reshape(-1, 3)
    return (t[:, 0] * nb + t[:, 2]) * nb + t[:, 1]          # (i, j, k)


def task_diff(tg, to, nb):
    """(only GPU, only oracle) triples, via sorted int64 keys (millions of triples)."""
    kg, ko = np.sort(keys(tg, nb)), np.sort(keys(to, nb))
    assert len(np.unique(kg)) == len(kg)
    if len(kg) == len(ko) and np.array_equal(kg, ko):
        return set(), set()

    def dec(k):
        return {(int(x // (nb * nb)), int(x % nb), int((x // nb) % nb)) for x in k}
    return dec(np.setdiff1d(kg, ko)), dec(np.setdiff1d(ko, kg))


def gpu_pattern(ctx, M, nb):
    L = nb.bit_length() - 1
    n2 = sp().spamm_level_norms2(ctx, M, L)
    bi, bj = np.nonzero(n2 > 0)
    assert len(bi) == M.nblocks            # every stored block has a non-zero norm
    return set(zip(bi.tolist(), bj.tolist()))


def compare_blocks(ctx, G, Go, corr_fn, nb, b, rng, full):
    """Pattern equality, then values over the union (all blocks or a sample)."""
    og = Go.block_coords()
    opat = set(zip(og[0].tolist(), og[1].tolist()))
    gpat = gpu_pattern(ctx, G, nb)
    union = sorted(gpat | opat)
    if not full:
        pick = rng.choice(len(union), size=min(1500, len(union)), replace=False)
        union = [union[i] for i in sorted(pick)]
    bi = np.array([u[0] for u in union], dtype=np.int32)
    bj = np.array([u[1] for u in union], dtype=np.int32)
    g, present = sp().spamm_get_blocks(ctx, G, bi, bj)
    gb = {u: g[t] for t, u in enumerate(union) if present[t]}
    ob = {}
    for u in union:
        o = Go.block(*u)
        if o is not None:
            ob[u] = o
    ob = corr_fn(ob)
    return gpat ^ opat, P.rel_union(gb, ob, set(union))


def check_step(ctx, Y, Z, n, b, tau, tau_s, rng, full, label):
    nb = n // b
    Yo, Zo = export(ctx, Y, n, b), export(ctx, Z, n, b)
    # pass 1 counts the triples, pass 2 (same inputs, deterministic) records them
    cnt = sp().VolumeSink(3)
    sp().spamm_ctx_set_volume_sink(ctx, cnt)
    Yn, Zn, t, st = sp().spamm_ns_step(ctx, Y, Z, tau, tau_s)
    sp().spamm_ctx_set_volume_sink(ctx, None)
    for M in (Yn, Zn):
        M.free()
    sink = sp().VolumeSink(3, ikj_cap=int(cnt.ntasks.sum()))
    sp().spamm_ctx_set_volume_sink(ctx, sink)
    Yn, Zn, t, st, H = sp().spamm_ns_step(ctx, Y, Z, tau, tau_s, want_h=True)
    sp().spamm_ctx_set_volume_sink(ctx, None)
    assert sink.complete() and list(sink.ntasks) == list(cnt.ntasks)
    Yno, Zno, Ho, to, counts, otasks = O.ns_step(Yo, Zo, tau, tau_s, want_tasks=True,
                                                 task_cap=int(cnt.ntasks.max()) + 1024)
    assert t == pytest.approx(to, abs=1e-12, rel=1e-12), (label, t, to)
    # task sets per product, modulo the window; the operands of each product
    operands = [(Zo, Yo, tau), (Yo, Ho, tau_s), (Ho, Zo, tau)]
    flips = []
    for p, (Ao, Bo, tp) in enumerate(operands):
        og, oo = task_diff(sink.tasks(p), otasks[p], nb)
        bad = P.outside_window(og | oo, Ao, Bo, tp)
        assert not bad, (label, p, len(bad), bad[:5])
        flips.append((og, oo))
        assert st[p]["tasks"] == sink.ntasks[p]
    if any(a or c for a, c in flips):
        print(f"{label}: flips inside the window {[(len(a), len(c)) for a, c in flips]}")
    # H = 1.5 I - 0.5 X: an X flip moves H_ij by -0.5 A_ik B_kj
    (xg, xo), (yg, yo), (zg, zo) = flips

    def corr_h(ob):
        c = P.flip_correct({}, Zo, Yo, xg, xo)
        out = dict(ob)
        for key, v in c.items():
            out[key] = out.get(key, np.zeros((b, b))) - 0.5 * v
        return out

    res = {}
    for name, G, Go, fn in (("H", H, Ho, corr_h),
                            ("Y'", Yn, Yno, lambda ob: P.flip_correct(ob, Yo, Ho, yg, yo)),
                            ("Z'", Zn, Zno, lambda ob: P.flip_correct(ob, Ho, Zo, zg, zo))):
        pdiff, err = compare_blocks(ctx, G, Go, fn, nb, b, rng, full)
        if not any(a or c for a, c in flips):
            assert not pdiff, (label, name, len(pdiff))
        assert err <= 1e-12, (label, name, err)
        res[name] = err
    norms = dict(Y=Yno.norm(), Z=Zno.norm(), Yg=sp().spamm_norm(ctx, Yn), Zg=sp().spamm_norm(ctx, Zn))
    return Yn, Zn, H, t, to, res, norms


def gpu_iterates(cfg, ctx, k_in, tau, tau_s):
    n, b = cfg.n, cfg.b
    _, (bi, bj, blocks) = si.make_input(cfg)
    dev = torch.device("cuda:0")
    S = sp().spamm_build_tree_blocks(ctx, n, b, *(torch.from_numpy(x).to(dev) for x in (bi, bj, blocks)))
    c = sp().spamm_power_scale(ctx, S, 100)
    Y = sp().spamm_ns_y0(ctx, S, c, cfg.mu)
    Z = sp().spamm_identity(ctx, n, b)
    S.free()
    for _ in range(k_in):
        Yn, Zn, _, _ = sp().spamm_ns_step(ctx, Y, Z, tau, tau_s)
        Y.free()
        Z.free()
        Y, Z = Yn, Zn
    return Y, Z


@pytest.mark.parametrize("cfg_name,k_in,tau_s_factor", [("C3", 8, None), ("C4", 2, None), ("C5", 1, None),
                                                         ("C5", 8, None)])
def test_lockstep_step_full_size(cfg_name, k_in, tau_s_factor):
    """C5 k = 8 is the bench's peak step (tau_s = .01 tau: ~2.7M Y' tasks)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = si.CONFIGS[cfg_name]
    tau = cfg.tau
    tau_s = tau * (cfg.tau_s_factor if tau_s_factor is None else tau_s_factor)
    ctx = sp().spamm_ctx_create(0)
    Y, Z = gpu_iterates(cfg, ctx, k_in, tau, tau_s)
    rng = np.random.default_rng(20261019)
    out = check_step(ctx, Y, Z, cfg.n, cfg.b, tau, tau_s, rng, full=(cfg_name == "C3"),
                     label=f"{cfg_name} k={k_in}")
    print(f"{cfg_name} k={k_in}: t={out[3]:.6e} errors {out[5]}")


def test_c5_tau_s_equal_tau_divergence_is_the_methods():
    """DESIGN.md reading L9: with tau_s = tau (the BASELINE.json literal), the GPU's C5 run
    leaves the basin at k = 10 (t_9 = 0.056, then ||Z|| doubles and t_10 ~ 2.6).  From the
    GPU's own Y_9, Z_9 the oracle's step must reproduce the jump (same task sets, Y_10,
    Z_10 norms and values), and from Y_10, Z_10 the same t_10: the divergence is the
    method's at this tau_s, not the kernels'."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = si.CONFIGS["C5"]
    tau = tau_s = cfg.tau
    ctx = sp().spamm_ctx_create(0)
    Y, Z = gpu_iterates(cfg, ctx, 9, tau, tau_s)
    rng = np.random.default_rng(9)
    Z9 = sp().spamm_norm(ctx, Z)
    Yn, Zn, H, t9, to9, res, norms = check_step(ctx, Y, Z, cfg.n, cfg.b, tau, tau_s, rng, False, "C5 k=9 tau_s=tau")
    assert norms["Zg"] == pytest.approx(norms["Z"], rel=1e-12)
    assert norms["Yg"] == pytest.approx(norms["Y"], rel=1e-12)
    growth = norms["Z"] / Z9
    print(f"C5 tau_s=tau k=9: t9 {t9:.6e} (oracle {to9:.6e}) ||Z10||/||Z9|| = {growth:.4f} "
          f"(GPU {norms['Zg'] / Z9:.4f}), errors {res}")
    assert growth > 2.0                      # the oracle's step doubles ||Z|| too
    H.free()
    Y.free()
    Z.free()
    # k = 10: t_10 from the GPU's Y_10, Z_10, on both sides
    Yo, Zo = export(ctx, Yn, cfg.n, cfg.b), export(ctx, Zn, cfg.n, cfg.b)
    Xo = O.multiply(Zo, Yo, tau)
    t10o = (cfg.n - Xo.trace()) / cfg.n
    del Xo
    X = sp().spamm_multiply(ctx, Zn, Yn, tau)
    t10g = (cfg.n - trace_of(ctx, X, cfg.n, cfg.b)) / cfg.n
    print(f"C5 tau_s=tau k=10: t10 GPU {t10g:.12e} oracle {t10o:.12e}")
    assert t10g == pytest.approx(t10o, rel=1e-12)
    assert t10o > 1.0                        # out of the basin: x(3-x)^2/4 diverges


def trace_of(ctx, X, n, b):
    nb = n // b
    idx = np.arange(nb, dtype=np.int32)
    blk, present = sp().spamm_get_blocks(ctx, X, idx, idx)
    return float(sum(np.trace(blk[i]) for i in range(nb) if present[i]))


def test_c3_free_run_full_iteration():
    """BASELINE.json configs[2] literally: C3, tau = tau_s = 1e-7, 30 fixed iterations
    (reading L15 for C1-C3), c from the oracle's power iteration.  All 90 task counts
    identical, t_k to 1e-12, Y and Z (every block, union of patterns) <= 1e-10: the
    kernel instantiation the bench times (b = 64) over a whole run, including the
    post-convergence fill-in of reading L15."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = si.CONFIGS["C3"]
    n, b = cfg.n, cfg.b
    _, (bi, bj, blocks) = si.make_input(cfg)
    So = O.OMat.from_blocks(n, b, bi, bj, blocks)
    c = O.power_scale(So, 100)
    ctx = sp().spamm_ctx_create(0)
    S = sp().spamm_build_tree_blocks(ctx, n, b, bi, bj, blocks)
    r = sp().spamm_ns_sqrt(ctx, S, cfg.tau, cfg.iters, tau_s=cfg.tau, scale=c)
    ro = O.ns_sqrt(So, cfg.tau, cfg.iters, tau_s=cfg.tau, scale=c)
    assert ro["rc"] == 0 and r["iters"] == ro["iters"] == cfg.iters
    counts = np.array([[p["tasks"] for p in k] for k in r["stats"]])
    np.testing.assert_allclose(r["t"], ro["t"], rtol=0, atol=1e-12)
    assert np.array_equal(counts, ro["counts"]), np.argwhere(counts != ro["counts"])[:5]
    for name, G, Go in (("Y", r["Y"], ro["Y"]), ("Z", r["Z"], ro["Z"])):
        err = P.rel_union(P.gpu_blocks(sp(), ctx, G), P.oracle_blocks(Go))
        print(f"C3 free run: {name} rel err {err:.3e}, {G.nblocks} blocks")
        assert err <= 1e-10, (name, err)
    print("C3 free run tasks per k:", counts.tolist())


@pytest.mark.parametrize("cfg_name", ["C3", "C5"])
def test_power_scale_full_size(cfg_name):
    """c ~ ||s||_2 (reading L12) at full size: the TMA-staged SpMV and the two-launch
    normalisation (n >= 65536) agree with the oracle's power iteration to 1e-12."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = si.CONFIGS[cfg_name]
    _, (bi, bj, blocks) = si.make_input(cfg)
    ctx = sp().spamm_ctx_create(0)
    S = sp().spamm_build_tree_blocks(ctx, cfg.n, cfg.b, bi, bj, blocks)
    c = sp().spamm_power_scale(ctx, S, 100)
    So = O.OMat.from_blocks(cfg.n, cfg.b, bi, bj, blocks)
    assert c == pytest.approx(O.power_scale(So, 100), rel=1e-12)
