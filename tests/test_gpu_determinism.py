"""Run-to-run determinism of the CUDA path (B200).

Every product is deterministic by construction (one CTA owns an output block and
accumulates its tasks in ascending k; fixed-order reductions), so repeated runs
must agree bitwise.  This caught a cross-proxy race in the leaf GEMM (generic
shared-memory reads of a stage vs. the TMA refill of that stage, fixed with
fence.proxy.async before the consumer's release), which corrupted ~1 product in
20 by a few ulps.  SPAMM_SELFCHECK=1 re-runs each cull and GEMM inside the
library and reports any bitwise mismatch on stderr."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

import spamm_inputs as si

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sp():
    import paper_1508_05856_b200 as m
    return m


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _hash(ctx, M):
    bi, bj, blk = sp().spamm_export_blocks(ctx, M)
    o = np.lexsort((bj, bi))
    return hashlib.sha1(bi[o].tobytes() + bj[o].tobytes() + blk[o].tobytes()).hexdigest()


@pytest.mark.parametrize("library_stream", [False, True])
def test_repeated_products_bitwise(gpu, library_stream):
    n, b = 4096, 64
    cfg = si.Config("t", "gauss", n, b, 1e-7, 30, sigma=0.8, shift=1e-3, seed=150805856, tau_min=1e-7)
    payload = si.make_input(cfg)[1]
    ctx = sp().spamm_ctx_create(0, library_stream=library_stream)
    S = sp().spamm_build_tree_blocks(ctx, n, b, *payload)
    Y, Z = sp().spamm_ns_y0(ctx, S, 11.0), sp().spamm_identity(ctx, n, b)
    for _ in range(4):
        Y, Z, _, _ = sp().spamm_ns_step(ctx, Y, Z, 1e-7, 1e-9)
    seen = {"X": set(), "Hs": set(), "Ys": set(), "H": set()}
    for _ in range(25):
        X = sp().spamm_multiply(ctx, Z, Y, 1e-7)
        seen["X"].add(_hash(ctx, X))
        X.free()
        Yn, Zn, _, _, _, H = sp().spamm_ns_step_map(ctx, Y, Z, 1e-7, 1e-9, scaled=True, want_h=True)
        seen["Hs"].add(_hash(ctx, H))
        seen["Ys"].add(_hash(ctx, Yn))
        for m in (Yn, Zn, H):
            m.free()
        Yn, Zn, _, _, H = sp().spamm_ns_step(ctx, Y, Z, 1e-7, 1e-9, want_h=True)
        seen["H"].add(_hash(ctx, H))
        for m in (Yn, Zn, H):
            m.free()
    assert all(len(v) == 1 for v in seen.values()), {k: len(v) for k, v in seen.items()}


def test_selfcheck_reports_no_mismatch(gpu):
    code = ("import sys; sys.path.insert(0, %r); import paper_1508_05856_b200 as sp, spamm_inputs as si\n"
            "c = si.CONFIGS['C2']; s = si.kms(c.n, c.rho); ctx = sp.spamm_ctx_create(0)\n"
            "S = sp.spamm_build_tree(ctx, s, c.b); r = sp.spamm_ns_sqrt(ctx, S, c.tau, 12)\n"
            "print('ok', r['iters'])\n") % ROOT
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "SPAMM_SELFCHECK": "1"})
    assert p.returncode == 0, p.stderr[-2000:]
    assert "ok 12" in p.stdout
    assert "SELFCHECK" not in p.stderr, p.stderr[-2000:]


def test_ns_sqrt_chained_equals_step_loop(gpu):
    """spamm_ns_sqrt enqueues each step's X cull before the previous step's closing fetch
    (and fuses the final unscale); a plain loop of spamm_ns_step does neither.  Same t_k
    sequence bitwise, same task counts, same iterates (up to the unscale's rounding)."""
    n, b, iters, c = 4096, 64, 6, 11.0
    cfg = si.Config("t", "gauss", n, b, 1e-7, 30, sigma=0.8, shift=1e-3, seed=150805856, tau_min=1e-7)
    payload = si.make_input(cfg)[1]
    ctx = sp().spamm_ctx_create(0)
    S = sp().spamm_build_tree_blocks(ctx, n, b, *payload)
    r = sp().spamm_ns_sqrt(ctx, S, 1e-7, iters, tau_s=1e-9, scale=c)
    Y, Z = sp().spamm_ns_y0(ctx, S, c), sp().spamm_identity(ctx, n, b)
    ts, counts = [], []
    for _ in range(iters):
        Yn, Zn, t, st = sp().spamm_ns_step(ctx, Y, Z, 1e-7, 1e-9)
        ts.append(t)
        counts.append([s["tasks"] for s in st])
        Y.free()
        Z.free()
        Y, Z = Yn, Zn
    assert np.array_equal(np.asarray(ts), r["t"])
    assert counts == [[s["tasks"] for s in k] for k in r["stats"]]
    f = np.sqrt(c)
    for M, ref, scale in ((r["Y"], Y, f), (r["Z"], Z, 1.0 / f)):
        bi, bj, blk = sp().spamm_export_blocks(ctx, M)
        ri, rj, rblk = sp().spamm_export_blocks(ctx, ref)
        o, q = np.lexsort((bj, bi)), np.lexsort((rj, ri))
        assert np.array_equal(bi[o], ri[q]) and np.array_equal(bj[o], rj[q])
        np.testing.assert_allclose(blk[o], rblk[q] * scale, rtol=4e-16, atol=0)


def test_allocators_agree_bitwise(gpu):
    """The library's own stream-ordered allocator (cudaMallocAsync: allocation nodes sit
    between the programmatically dependent launches) and PyTorch's caching allocator give
    the same NS run bitwise."""
    c = si.CONFIGS["C2"]
    s = si.kms(c.n, c.rho)
    out = []
    for torch_alloc in (True, False):
        ctx = sp().spamm_ctx_create(0, torch_allocator=torch_alloc)
        S = sp().spamm_build_tree(ctx, s, c.b)
        r = sp().spamm_ns_sqrt(ctx, S, c.tau, 10)
        out.append((r["t"].copy(), _hash(ctx, r["Y"]), _hash(ctx, r["Z"]), r["c"]))
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1:] == out[1][1:]


def test_ab_switches_bitwise():
    """The A/B switches change stream and launch ordering only: SPAMM_CONCURRENT_CULL=0/1
    (the Z' cull on the side stream or after the Y' cull), SPAMM_PDL=0/1 (programmatic
    dependent launch or plain stream order), SPAMM_CULL_SMALL=0/1 (the single-CTA
    query or the multi-kernel chain) and SPAMM_CULL_FLAT=0/1 (the flat small-problem query
    or the level walk), SPAMM_GRAPH_PAIR=0/1 (the captured step's Y' and Z' GEMMs and
    pyramids grouped or not) and SPAMM_GRAPH_SIDE_CLEAR=0/1 give the same NS run bitwise
    (t_k, Y, Z, every product's task, segment and per-level survivor counts)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_1508_05856_b200 as sp, spamm_inputs as si\n"
            "c = si.CONFIGS['C2']; s = si.kms(c.n, c.rho); ctx = sp.spamm_ctx_create(0)\n"
            "S = sp.spamm_build_tree(ctx, s, c.b); r = sp.spamm_ns_sqrt(ctx, S, c.tau, 12)\n"
            "h = hashlib.sha1(r['t'].tobytes() + repr([[p['tasks'], p['segments'], p['level_survivors']]"
            " for k in r['stats'] for p in k]).encode())\n"
            "for M in (r['Y'], r['Z']):\n"
            "    bi, bj, blk = sp.spamm_export_blocks(ctx, M); o = np.lexsort((bj, bi))\n"
            "    h.update(bi[o].tobytes() + bj[o].tobytes() + blk[o].tobytes())\n"
            "print('hash', h.hexdigest())\n") % ROOT
    seen = {}
    for conc, pdl, small, flat in (("0", "0", "1", "0"), ("0", "1", "1", "0"), ("1", "0", "1", "0"),
                                   ("1", "1", "1", "0"), ("1", "1", "1", "1"), ("1", "1", "0", "0"),
                                   ("0", "0", "0", "0"), ("0", "0", "1", "1")):
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env={**os.environ, "SPAMM_CONCURRENT_CULL": conc, "SPAMM_PDL": pdl,
                                "SPAMM_CULL_SMALL": small, "SPAMM_CULL_FLAT": flat})
        assert p.returncode == 0, p.stderr[-2000:]
        seen[(conc, pdl, small, flat)] = [l for l in p.stdout.splitlines() if l.startswith("hash")][-1]
    # the captured step's grouped Y'/Z' GEMM + pyramids and its side-stream pattern clearing
    for pair, side in (("0", "1"), ("1", "0"), ("0", "0")):
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env={**os.environ, "SPAMM_GRAPH_PAIR": pair, "SPAMM_GRAPH_SIDE_CLEAR": side})
        assert p.returncode == 0, p.stderr[-2000:]
        seen[("pair", pair, side)] = [l for l in p.stdout.splitlines() if l.startswith("hash")][-1]
    assert len(set(seen.values())) == 1, seen


@pytest.mark.parametrize("case", ["C1", "C2", "gauss4096"])
def test_graph_replay_equals_host_driven(case):
    """Small runs replay a captured, device-driven dual step (SPAMM_GRAPH=1, the default
    when the worst-case workspace fits): same kernels and orders as the host-driven loop
    (SPAMM_GRAPH=0), so t_k, every product's counts and Y, Z are bitwise equal.  A second
    run on the same context replays the cached graphs and must agree too."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    setup = {
        "C1": "c = si.CONFIGS['C1']; S = sp.spamm_build_tree(ctx, si.kms(c.n, c.rho), c.b); tau, it = c.tau, c.iters\n",
        "C2": "c = si.CONFIGS['C2']; S = sp.spamm_build_tree(ctx, si.kms(c.n, c.rho), c.b); tau, it = c.tau, c.iters\n",
        "gauss4096": ("c = si.Config('t', 'gauss', 4096, 64, 1e-7, 30, sigma=0.8, shift=1e-3, seed=150805856, "
                      "tau_min=1e-7); S = sp.spamm_build_tree_blocks(ctx, 4096, 64, *si.make_input(c)[1]); "
                      "tau, it = 1e-7, 20\n"),
    }[case]
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_1508_05856_b200 as sp, spamm_inputs as si\n"
            "ctx = sp.spamm_ctx_create(0)\n" + setup +
            "for rep in range(2):\n"
            "    r = sp.spamm_ns_sqrt(ctx, S, tau, it)\n"
            "    h = hashlib.sha1(r['t'].tobytes() + repr([[p['tasks'], p['segments'], p['level_survivors']]"
            " for k in r['stats'] for p in k]).encode())\n"
            "    for M in (r['Y'], r['Z']):\n"
            "        bi, bj, blk = sp.spamm_export_blocks(ctx, M); o = np.lexsort((bj, bi))\n"
            "        h.update(bi[o].tobytes() + bj[o].tobytes() + blk[o].tobytes())\n"
            "    print('hash', r['iters'], h.hexdigest())\n") % ROOT
    out = {}
    for gm in ("0", "1"):
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900,
                           env={**os.environ, "SPAMM_GRAPH": gm})
        assert p.returncode == 0, p.stderr[-3000:]
        out[gm] = [l for l in p.stdout.splitlines() if l.startswith("hash")]
        assert len(out[gm]) == 2 and out[gm][0] == out[gm][1], out[gm]
    assert out["0"][0] == out["1"][0], out
