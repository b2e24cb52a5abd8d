"""Parity at BASELINE.json's full sizes, in the configuration bench.py times (B200).

One dual NS step in lockstep at the configs' full n: the GPU produces the input
iterates (Y_k, Z_k) of the bench run (same tau, tau_s, seeded input), they are
exported, and the CPU oracle runs the same step from them (Eq. cannonical in the
north_star form, Eq. newspamm products).  Compared (north_star bars, BJ:5):
  * the three task counts: identical (a flip would have to sit within 1e-12 of the
    threshold; none is expected among ~1e6 tests);
  * t_k to 1e-12 absolute;
  * H, Y', Z' on a seeded sample of output blocks: relative Frobenius <= 1e-12.
The oracle runs on the box's host cores (~1e12 flop per C5 step).
"""
import math

import numpy as np
import pytest

import oracle as O
import spamm_inputs as si

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def sp():
    import paper_1508_05856_b200 as m
    return m


def export(ctx, M, n, b):
    bi, bj, blk = sp().spamm_export_blocks(ctx, M)
    return O.OMat.from_blocks(n, b, bi, bj, blk), (bi, bj, blk)


def sampled_rel(ctx, G, Go_blocks_fn, n, b, coords, rng, k=1500):
    pick = rng.choice(len(coords[0]), size=min(k, len(coords[0])), replace=False)
    bi, bj = coords[0][pick].astype(np.int32), coords[1][pick].astype(np.int32)
    g, present = sp().spamm_get_blocks(ctx, G, bi, bj)
    num = den = 0.0
    for t, (I, J) in enumerate(zip(bi, bj)):
        o = Go_blocks_fn(int(I), int(J))
        o = np.zeros((b, b)) if o is None else o
        num += np.sum((g[t] - o) ** 2)
        den += np.sum(o ** 2)
    return math.sqrt(num / den), int(present.sum())


@pytest.mark.parametrize("cfg_name,k_in", [("C3", 8), ("C4", 2), ("C5", 1)])
def test_lockstep_step_full_size(cfg_name, k_in):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cfg = si.CONFIGS[cfg_name]
    n, b, tau = cfg.n, cfg.b, cfg.tau
    tau_s = tau * cfg.tau_s_factor
    _, (bi, bj, blocks) = si.make_input(cfg)
    ctx = sp().spamm_ctx_create(0)
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
    Yo, _ = export(ctx, Y, n, b)
    Zo, _ = export(ctx, Z, n, b)
    Yn, Zn, t, st, H = sp().spamm_ns_step(ctx, Y, Z, tau, tau_s, want_h=True)
    Yno, Zno, Ho, to, cnt = O.ns_step(Yo, Zo, tau, tau_s)
    assert [s["tasks"] for s in st] == list(cnt), (cfg_name, [s["tasks"] for s in st], list(cnt))
    assert t == pytest.approx(to, abs=1e-12)
    rng = np.random.default_rng(20261019)
    for G, Go in ((H, Ho), (Yn, Yno), (Zn, Zno)):
        coords = Go.block_coords()
        assert G.nblocks == Go.nblocks()
        err, present = sampled_rel(ctx, G, Go.block, n, b, coords, rng)
        assert present == min(1500, len(coords[0]))
        assert err <= 1e-12, (cfg_name, err)


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
