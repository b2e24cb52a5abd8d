"""GPU (B200) parity of the CUDA path, through the C ABI, against the CPU oracle.

Bars (BASELINE.json north_star, BJ:5):
  * surviving task sets identical except triples whose norm product lies within
    1e-12 relative of the threshold;
  * relative Frobenius error of each product <= 1e-12;
  * relative Frobenius error of Y and Z after the full iteration <= 1e-10.
Leaf norms / pyramid: <= 1e-14 relative (different but fixed summation orders).
"""
import math

import numpy as np
import pytest

import _parity as P
import oracle as O
import spamm_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1508_05856_b200 as sp
    return sp.spamm_ctx_create(0)


def sp():
    import paper_1508_05856_b200 as m
    return m


def decaying(n, rate, seed, zero_frac=0.0):
    r = np.random.default_rng(seed)
    i = np.arange(n)
    d = np.abs(i[:, None] - i[None, :])
    m = np.exp(-rate * d) * r.standard_normal((n, n))
    return m


def gpu_to_oracle(ctx, M):
    """Copy a GPU quadtree to an oracle tree (present blocks only)."""
    n, b, _ = M.info()
    nb = n // b
    L = nb.bit_length() - 1
    n2 = sp().spamm_level_norms2(ctx, M, L)
    bi, bj = np.nonzero(n2 > 0)
    blocks, pres = sp().spamm_get_blocks(ctx, M, bi, bj)
    assert pres.all()
    return O.OMat.from_blocks(n, b, bi.astype(np.int32), bj.astype(np.int32), blocks)


def build_pair(ctx, kind, payload, b, n):
    if kind == "dense":
        d = torch.from_numpy(payload).cuda()
        return sp().spamm_build_tree(ctx, d, b), O.OMat.from_dense(payload, b)
    bi, bj, blocks = payload
    G = sp().spamm_build_tree_blocks(ctx, n, b, torch.from_numpy(bi).cuda(),
                                     torch.from_numpy(bj).cuda(), torch.from_numpy(blocks).cuda())
    return G, O.OMat.from_blocks(n, b, bi, bj, blocks)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def check_product(ctx, A, Ao, B, Bo, tau, vals_tol=1e-12, trans_a=False):
    """SURVEY.md §8(c) protocol for one product: the task set equals the oracle's except
    within the 1e-12 window; the values, flip-corrected, agree to vals_tol over the union
    of both sides' blocks; the epilogue's leaf norms agree with the corrected blocks'."""
    mul = sp().spamm_multiply_t if trans_a else sp().spamm_multiply
    C, st = mul(ctx, A, B, tau, want_stats=True)
    tg = sp().spamm_export_tasks(ctx)
    Co, to = O.multiply(Ao, Bo, tau, want_tasks=True, trans_a=trans_a)
    Al = O.transpose(Ao) if trans_a else Ao
    sg, so = P.triples(tg), P.triples(to)
    assert len(sg) == len(tg) == st["tasks"]
    only_g, only_o = sg - so, so - sg
    bad = P.outside_window(only_g | only_o, Al, Bo, tau)
    assert not bad, f"{len(bad)} task flips outside the window: {bad[:5]}"
    # tasks grouped by output block (Morton order), k ascending inside a segment
    if len(tg):
        ij = tg[:, 0].astype(np.int64) * (1 << 20) + tg[:, 2]
        change = np.nonzero(np.diff(ij))[0]
        starts = np.r_[0, change + 1]
        assert len(np.unique(ij)) == len(starts) == st["segments"]
        for s0, s1 in zip(starts, np.r_[starts[1:], len(tg)]):
            assert np.all(np.diff(tg[s0:s1, 1]) > 0)
    gb = P.gpu_blocks(sp(), ctx, C)
    ob = P.flip_correct(P.oracle_blocks(Co), Al, Bo, only_g, only_o)
    assert P.rel_union(gb, ob) <= vals_tol
    # every stored GPU block has a non-zero epilogue norm, and the norms match
    L = (Ao.n // Ao.b).bit_length() - 1
    n2 = sp().spamm_level_norms2(ctx, C, L)
    ref = np.zeros_like(n2)
    for (I, J), o in ob.items():
        ref[I, J] = np.sqrt(np.sum(o * o))
    assert set(zip(*np.nonzero(n2 > 0))) == set(gb)
    np.testing.assert_allclose(np.sqrt(n2), ref, rtol=1e-12, atol=1e-300)
    return C, Co


# ------------------------------------------------------------------ tree
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_build_norms(ctx, cfg):
    c = si.CONFIGS[cfg]
    kind, payload = si.make_input(c)
    G, Og = build_pair(ctx, kind, payload, c.b, c.n)
    L = (c.n // c.b).bit_length() - 1
    for lev in sorted({0, 1, L // 2, L - 1, L}):
        g = sp().spamm_level_norms2(ctx, G, lev)
        np.testing.assert_allclose(np.sqrt(g), Og.level_norms(lev), rtol=1e-14, atol=0)
    assert sp().spamm_norm(ctx, G) == pytest.approx(Og.norm(), rel=1e-14)
    assert G.nblocks == Og.nblocks()
    if c.n <= 4096:
        d = sp().spamm_to_dense(ctx, G).cpu().numpy()
        assert np.array_equal(d, Og.to_dense())


def test_build_host_pointer_and_ld(ctx):
    m = decaying(256, 0.1, 5)
    m[16:32, 64:80] = 0.0
    big = np.zeros((256, 300))
    big[:, :256] = m
    G = sp().spamm_build_tree(ctx, big[:, :256].copy(), 16)
    assert np.array_equal(sp().spamm_to_dense(ctx, G, device=False), m)
    Gt = sp().spamm_build_tree(ctx, torch.from_numpy(big).cuda()[:, :256].contiguous(), 16)
    assert np.array_equal(sp().spamm_to_dense(ctx, Gt).cpu().numpy(), m)
    assert G.nblocks == 255


# --------------------------------------------------------------- product
def test_tiebreak_and_partial_cull_exact(ctx):
    A = np.ones((32, 32))
    G, Og = build_pair(ctx, "dense", A, 16, 32)
    C = sp().spamm_multiply(ctx, G, G, 0.25)
    assert len(sp().spamm_export_tasks(ctx)) == 8
    assert np.all(sp().spamm_to_dense(ctx, C).cpu().numpy() == 32.0)
    C = sp().spamm_multiply(ctx, G, G, np.nextafter(0.25, 1))
    assert len(sp().spamm_export_tasks(ctx)) == 0
    assert np.all(sp().spamm_to_dense(ctx, C).cpu().numpy() == 0.0)
    P = np.ones((16, 16)) / 16
    e = 1 / 8
    A = np.block([[P, e * P], [e * P, P]])
    G, _ = build_pair(ctx, "dense", A, 16, 32)
    C = sp().spamm_multiply(ctx, G, G, 1 / 32)
    t = {tuple(x) for x in sp().spamm_export_tasks(ctx)}
    assert t == {(0, 0, 0), (0, 0, 1), (0, 1, 1), (1, 0, 0), (1, 1, 0), (1, 1, 1)}
    assert np.array_equal(sp().spamm_to_dense(ctx, C).cpu().numpy(),
                          np.block([[P, P / 4], [P / 4, P]]))


@pytest.mark.parametrize("n,b", [(64, 64), (128, 16), (512, 16), (1024, 32), (2048, 64), (4096, 64)])
@pytest.mark.parametrize("tau", [0.0, 1e-8, 1e-4])
def test_multiply_random(ctx, n, b, tau):
    a = decaying(n, 20.0 / n, n + b)
    c = decaying(n, 30.0 / n, n + 2 * b)
    nb = n // b
    if nb >= 4:   # ragged pattern: absent blocks
        a[:b, 2 * b:3 * b] = 0.0
        c[(nb - 1) * b:, :b] = 0.0
    A, Ao = build_pair(ctx, "dense", a, b, n)
    B, Bo = build_pair(ctx, "dense", c, b, n)
    C, Co = check_product(ctx, A, Ao, B, Bo, tau)
    if tau == 0.0:
        ref = a @ c
        assert rel(sp().spamm_to_dense(ctx, C).cpu().numpy(), ref) <= 1e-13


@pytest.mark.parametrize("b", [64, 32, 16])
@pytest.mark.parametrize("band", [0, 1])
def test_multiply_short_segments(ctx, b, band):
    """Block-(tri)diagonal operands with nb = 1024 block rows: every output block has 1
    (band 0) or 1-3 (band 1) leaf tasks, so each CTA of the persistent GEMM hands the
    epilogue tile from its consumer warps to its epilogue warps after every task or two,
    ~7-20 times per launch.  Values, norms and task order go through check_product."""
    nb = 1024
    n = nb * b
    r = np.random.default_rng(b + band)
    bi, bj = [], []
    for I in range(nb):
        for J in range(max(0, I - band), min(nb, I + band + 1)):
            bi.append(I)
            bj.append(J)
    bi = np.array(bi, dtype=np.int32)
    bj = np.array(bj, dtype=np.int32)
    A, Ao = build_pair(ctx, "blocks", (bi, bj, r.standard_normal((len(bi), b, b))), b, n)
    B, Bo = build_pair(ctx, "blocks", (bi, bj, r.standard_normal((len(bi), b, b))), b, n)
    C, st = sp().spamm_multiply(ctx, A, B, 0.0, want_stats=True)
    assert st["segments"] == (nb if band == 0 else 5 * nb - 6)   # |I - J| <= 2 * band
    check_product(ctx, A, Ao, B, Bo, 0.0)


def test_multiply_degenerate(ctx):
    z = np.zeros((128, 128))
    Z, Zo = build_pair(ctx, "dense", z, 16, 128)
    a = decaying(128, 0.1, 1)
    A, Ao = build_pair(ctx, "dense", a, 16, 128)
    C = sp().spamm_multiply(ctx, Z, A, 0.0)
    assert C.nblocks == 0 and len(sp().spamm_export_tasks(ctx)) == 0
    C = sp().spamm_multiply(ctx, A, A, 1.0 + 1e-15)
    assert C.nblocks == 0
    with pytest.raises(sp().SpammError) as e:
        sp().spamm_multiply(ctx, A, A, -1.0)
    assert e.value.code == 1
    B16, _ = build_pair(ctx, "dense", decaying(256, 0.1, 2), 16, 256)
    with pytest.raises(sp().SpammError) as e:
        sp().spamm_multiply(ctx, A, B16, 0.0)
    assert e.value.code == 2
    # n == b: a single leaf (L = 0)
    s1 = decaying(64, 0.1, 3)
    S1, S1o = build_pair(ctx, "dense", s1, 64, 64)
    check_product(ctx, S1, S1o, S1, S1o, 0.0)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_multiply_config_operands(ctx, cfg):
    """s (x)_tau s and I (x)_tau s on the config inputs."""
    c = si.CONFIGS[cfg]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    check_product(ctx, S, So, S, So, c.tau)
    I = sp().spamm_identity(ctx, c.n, c.b)
    Io = O.OMat.identity(c.n, c.b)
    check_product(ctx, I, Io, S, So, c.tau)


def test_multiply_c3_full_size(ctx):
    """C3 operands at full size (n = 16384, b = 64): Y0 (x)_tau Y0, sampled blocks."""
    c = si.CONFIGS["C3"]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    check_product(ctx, S, So, S, So, c.tau)


# -------------------------------------------------------------- NS
def test_power_scale(ctx):
    for cfg in ("C1", "C2"):
        c = si.CONFIGS[cfg]
        kind, payload = si.make_input(c)
        S, So = build_pair(ctx, kind, payload, c.b, c.n)
        assert sp().spamm_power_scale(ctx, S, 100) == pytest.approx(O.power_scale(So, 100), rel=1e-12)


@pytest.mark.parametrize("b", [64, 32, 16])
@pytest.mark.parametrize("case", ["sym", "sym_holes", "asym_values", "asym_pattern"])
def test_power_scale_symmetric_and_fallback(ctx, case, b):
    """b = 64: a bitwise-symmetric s takes the upper-half SpMV (column parts of the
    off-diagonal blocks), anything else the full SpMV; b < 64: the register SpMV.  All
    match the oracle's plain power iteration (reading L12).  Holes: absent off-diagonal
    blocks in a symmetric pattern, and an empty block row tail."""
    n = 2048                            # nb = 32 / 64 / 128: several units per row, ragged quarters
    m = np.abs(decaying(n, 0.01, 7))
    m = m + m.T
    nb = n // b
    if case in ("sym_holes", "asym_pattern"):
        r = np.random.default_rng(3)
        for I in range(nb):
            for J in range(I + 1, nb):
                if r.random() < 0.4:
                    m[I * b:(I + 1) * b, J * b:(J + 1) * b] = 0
                    if case == "sym_holes":
                        m[J * b:(J + 1) * b, I * b:(I + 1) * b] = 0
    if case == "asym_values":
        m[5, 700] *= 1.0 + 2.0 ** -40
    S, So = build_pair(ctx, "dense", m, b, n)
    assert sp().spamm_power_scale(ctx, S, 100) == pytest.approx(O.power_scale(So, 100), rel=1e-12)


def test_ns_step_lockstep(ctx):
    """One dual step from identical inputs: H, t, Y', Z' and the three task counts."""
    c = si.CONFIGS["C2"]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    cs = O.power_scale(So)
    Y = sp().spamm_ns_y0(ctx, S, cs)
    Z = sp().spamm_identity(ctx, c.n, c.b)
    for k in range(6):
        Yo, Zo = gpu_to_oracle(ctx, Y), gpu_to_oracle(ctx, Z)
        Yn, Zn, t, st, H = sp().spamm_ns_step(ctx, Y, Z, c.tau, want_h=True)
        Yno, Zno, Ho, to, cnt = O.ns_step(Yo, Zo, c.tau)
        assert [s["tasks"] for s in st] == list(cnt)
        assert t == pytest.approx(to, abs=1e-13)
        assert rel(gpu_to_oracle(ctx, H).to_dense(), Ho.to_dense()) <= 1e-12
        assert rel(gpu_to_oracle(ctx, Yn).to_dense(), Yno.to_dense()) <= 1e-12
        assert rel(gpu_to_oracle(ctx, Zn).to_dense(), Zno.to_dense()) <= 1e-12
        Y, Z = Yn, Zn


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_ns_free_run(ctx, cfg):
    """Full iteration at the config's tau and iters: Y, Z within 1e-10 of the oracle."""
    c = si.CONFIGS[cfg]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    cs = O.power_scale(So)
    r = sp().spamm_ns_sqrt(ctx, S, c.tau, c.iters, scale=cs)
    ro = O.ns_sqrt(So, c.tau, c.iters, scale=cs)
    Yg, Zg = gpu_to_oracle(ctx, r["Y"]), gpu_to_oracle(ctx, r["Z"])
    assert rel(Yg.to_dense(), ro["Y"].to_dense()) <= 1e-10
    assert rel(Zg.to_dense(), ro["Z"].to_dense()) <= 1e-10
    np.testing.assert_allclose(r["t"], ro["t"], rtol=0, atol=1e-12)
    counts = np.array([[p["tasks"] for p in k] for k in r["stats"]])
    assert np.array_equal(counts, ro["counts"])


def test_ns_tau0_closed_form(ctx):
    """tau = 0: Z.Z equals the KMS tridiagonal inverse; Y.Z = I."""
    n, b, rho = 1024, 32, 0.5
    s = si.kms(n, rho)
    S = sp().spamm_build_tree(ctx, torch.from_numpy(s).cuda(), b)
    r = sp().spamm_ns_sqrt(ctx, S, 0.0, 25)
    Y = sp().spamm_to_dense(ctx, r["Y"]).cpu().numpy()
    Z = sp().spamm_to_dense(ctx, r["Z"]).cpu().numpy()
    k = 1 / (1 - rho ** 2)
    inv = np.diag(np.full(n, (1 + rho ** 2) * k))
    inv[0, 0] = inv[-1, -1] = k
    inv += np.diag(np.full(n - 1, -rho * k), 1) + np.diag(np.full(n - 1, -rho * k), -1)
    assert rel(Z @ Z, inv) <= 1e-12
    assert np.linalg.norm(Y @ Z - np.eye(n)) / math.sqrt(n) <= 1e-13


def test_ns_mu_shift(ctx):
    c = si.CONFIGS["C1"]
    s = si.kms(c.n, 0.7)
    S, So = build_pair(ctx, "dense", s, c.b, c.n)
    cs = O.power_scale(So)
    r = sp().spamm_ns_sqrt(ctx, S, 1e-8, 30, mu=1e-2, scale=cs)
    ro = O.ns_sqrt(So, 1e-8, 30, mu=1e-2, scale=cs)
    assert rel(gpu_to_oracle(ctx, r["Y"]).to_dense(), ro["Y"].to_dense()) <= 1e-10
    assert rel(gpu_to_oracle(ctx, r["Z"]).to_dense(), ro["Z"].to_dense()) <= 1e-10


# ------------------------------------------- scaled / stabilised map (§8(f) f1)
def test_ns_scaled_lockstep(ctx):
    """Scaled + stabilised map from identical inputs: t_k, (alpha, eps), H,
    Y', Z' and the task counts against the oracle."""
    c = si.CONFIGS["C2"]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    cs = O.power_scale(So)
    Y = sp().spamm_ns_y0(ctx, S, cs)
    Z = sp().spamm_identity(ctx, c.n, c.b)
    for k in range(6):
        Yo, Zo = gpu_to_oracle(ctx, Y), gpu_to_oracle(ctx, Z)
        Yn, Zn, t, st, (a, e), H = sp().spamm_ns_step_map(ctx, Y, Z, c.tau, scaled=True, want_h=True)
        Yno, Zno, Ho, to, cnt = O.ns_step(Yo, Zo, c.tau, scaled=True)
        assert t == pytest.approx(to, abs=1e-13)
        assert a == pytest.approx(O.alpha(to), rel=1e-12) and e == pytest.approx(O.eps(to), rel=1e-10, abs=1e-300)
        assert [s["tasks"] for s in st] == list(cnt)
        assert rel(gpu_to_oracle(ctx, H).to_dense(), Ho.to_dense()) <= 1e-12
        assert rel(gpu_to_oracle(ctx, Yn).to_dense(), Yno.to_dense()) <= 1e-12
        assert rel(gpu_to_oracle(ctx, Zn).to_dense(), Zno.to_dense()) <= 1e-12
        Y, Z = Yn, Zn


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_ns_scaled_free_run_and_t_stop(ctx, cfg):
    c = si.CONFIGS[cfg]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    cs = O.power_scale(So)
    r = sp().spamm_ns_sqrt(ctx, S, c.tau, c.iters, scale=cs, scaled=True, t_stop=1e-9)
    ro = O.ns_sqrt(So, c.tau, c.iters, scale=cs, scaled=True, t_stop=1e-9)
    assert r["iters"] == ro["iters"] < c.iters
    assert rel(gpu_to_oracle(ctx, r["Y"]).to_dense(), ro["Y"].to_dense()) <= 1e-10
    assert rel(gpu_to_oracle(ctx, r["Z"]).to_dense(), ro["Z"].to_dense()) <= 1e-10
    np.testing.assert_allclose(r["t"], ro["t"], rtol=0, atol=1e-12)
    counts = np.array([[p["tasks"] for p in k] for k in r["stats"]])
    assert np.array_equal(counts, ro["counts"])


# ------------------------------------------- single channel (§8(f) f2)
@pytest.mark.parametrize("n,b", [(128, 16), (1024, 32), (2048, 64)])
@pytest.mark.parametrize("tau", [0.0, 1e-6])
def test_multiply_transposed(ctx, n, b, tau):
    """A^T (x)_tau B: task set (modulo the window) and values vs the oracle's transposed tree."""
    a = decaying(n, 20.0 / n, n + 7 * b)
    c = decaying(n, 30.0 / n, n + 9 * b)
    a[:b, 2 * b:3 * b] = 0.0
    A, Ao = build_pair(ctx, "dense", a, b, n)
    B, Bo = build_pair(ctx, "dense", c, b, n)
    Cg, _ = check_product(ctx, A, Ao, B, Bo, tau, trans_a=True)
    if tau == 0.0:
        assert rel(sp().spamm_to_dense(ctx, Cg).cpu().numpy(), a.T @ c) <= 1e-13


@pytest.mark.parametrize("cfg,scaled", [("C1", False), ("C2", False), ("C2", True)])
def test_ns_single_channel_free_run(ctx, cfg, scaled):
    """Single channel full run vs the oracle: Y, Z <= 1e-10, t_k, task counts."""
    c = si.CONFIGS[cfg]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    cs = O.power_scale(So)
    tau_s = 0.01 * c.tau
    r = sp().spamm_ns_sqrt_single(ctx, S, c.tau, c.iters, tau_s=tau_s, scale=cs, scaled=scaled, t_stop=1e-9)
    ro = O.ns_sqrt_single(So, c.tau, c.iters, tau_s=tau_s, scale=cs, scaled=scaled, t_stop=1e-9)
    assert r["iters"] == ro["iters"]
    np.testing.assert_allclose(r["t"], ro["t"], rtol=0, atol=1e-12)
    counts = np.array([[p["tasks"] for p in k] for k in r["stats"]])
    assert np.array_equal(counts, ro["counts"])
    assert rel(gpu_to_oracle(ctx, r["Y"]).to_dense(), ro["Y"].to_dense()) <= 1e-10
    assert rel(gpu_to_oracle(ctx, r["Z"]).to_dense(), ro["Z"].to_dense()) <= 1e-10


def test_task_distance_histogram(ctx):
    """Lensing instrumentation (§8(f) f4): the histogram of max(|i-j|,|i-k|,|j-k|) over the
    surviving triples equals the one computed from the oracle's task list (exact ints)."""
    c = si.CONFIGS["C2"]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    sp().spamm_multiply(ctx, S, S, c.tau)
    h = sp().spamm_task_distance_hist(ctx, 200)
    _, to = O.multiply(So, So, c.tau, want_tasks=True)
    d = np.max(np.abs(np.stack([to[:, 0] - to[:, 2], to[:, 0] - to[:, 1], to[:, 2] - to[:, 1]])), axis=0)
    ref = np.bincount(np.minimum(d, 199), minlength=200)
    assert np.array_equal(h, ref)
    assert h.sum() == len(to)


# ------------------------------------- regularised product representation (§8(f) f3)
def test_regularized_factor_parity(ctx):
    """3 slices (mu = .1, .01, .001) on the C2 matrix (kappa 361) at tau0 = 1e-6, tau1 = 1e-8:
    G vs the oracle (1e-10), same per-slice iteration counts, and G^T (s + c mu_m I) G ~ I."""
    c = si.CONFIGS["C2"]
    s = si.kms(c.n, c.rho)
    S, So = build_pair(ctx, "dense", s, c.b, c.n)
    cs = O.power_scale(So)
    mus = [1e-1, 1e-2, 1e-3]
    r = sp().spamm_regularized_factor(ctx, S, 1e-6, 1e-8, mus, 40, t_stop=1e-9, scale=cs)
    ro = O.regularized_factor(So, 1e-6, 1e-8, mus, 40, t_stop=1e-9, scale=cs)
    assert list(r["slice_iters"]) == list(ro["slice_iters"])
    G = gpu_to_oracle(ctx, r["G"]).to_dense()
    assert rel(G, ro["G"].to_dense()) <= 1e-10
    sm = s + cs * mus[-1] * np.eye(c.n)
    # an approximate inverse factor: the paper's slices carry "a numerical resolution of
    # approximately one digit"; here ~2e-3 per unit of the spectrum
    assert np.linalg.norm(G.T @ sm @ G - np.eye(c.n)) / math.sqrt(c.n) <= 1e-2


def test_ns_nonfinite_reported(ctx):
    """a run that diverges (scale far below ||s||_2, so the NS map leaves its
    basin: x(3-x)^2/4 explodes for x > 5) returns SPAMM_ENOTFINITE; the oracle reports the
    failure too."""
    c = si.CONFIGS["C1"]
    s = si.kms(c.n, c.rho)
    S, So = build_pair(ctx, "dense", s, c.b, c.n)
    bad = O.power_scale(So) / 8.0
    with pytest.raises(sp().SpammError) as e:
        sp().spamm_ns_sqrt(ctx, S, c.tau, 25, scale=bad)
    assert e.value.code == 6
    ro = O.ns_sqrt(So, c.tau, 25, scale=bad)
    assert ro["rc"] != 0        # non-finite t_k or root norm
    # the context stays usable after the failure
    r = sp().spamm_ns_sqrt(ctx, S, c.tau, 5, scale=O.power_scale(So))
    assert np.all(np.isfinite(r["t"]))


@pytest.mark.parametrize("cfg", ["C3", "C2", "C1"])
def test_power_scale_sym_and_full_paths_bitwise(ctx, cfg):
    """For a symmetric s the upper-triangle SpMV and the full SpMV (used when s is not
    symmetric, and by every rank of a row partition) compute the lower blocks' share in
    the same order, so c is bitwise the same (what keeps the row-partitioned run bitwise
    equal to the single-device run).  C3: the TMA ring (b = 64); C2 / C1: the per-block
    kernel (b = 32 / 16); the zig-zag schedule must not change c either."""
    code = ("import sys; sys.path.insert(0, %r); import paper_1508_05856_b200 as sp, spamm_inputs as si, torch\n"
            "c = si.CONFIGS[%r]; kind, p = si.make_input(c); ctx = sp.spamm_ctx_create(0)\n"
            "S = (sp.spamm_build_tree_blocks(ctx, c.n, c.b, *(torch.from_numpy(x).cuda() for x in p))\n"
            "     if kind == 'blocks' else sp.spamm_build_tree(ctx, torch.from_numpy(p).cuda(), c.b))\n"
            "print(repr(sp.spamm_power_scale(ctx, S, 100)))\n")
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = []
    for env in ({"SPAMM_SPMV_SYM": "1"}, {"SPAMM_SPMV_SYM": "0"}, {"SPAMM_SPMV_ZIGZAG": "0"}):
        p = subprocess.run([sys.executable, "-c", code % (root, cfg)], capture_output=True, text=True, timeout=600,
                           env={**os.environ, **env})
        assert p.returncode == 0, p.stderr[-2000:]
        out.append(p.stdout.strip().splitlines()[-1])
    assert out[0] == out[1] == out[2], out


def test_volume_sink_whole_run_matches_oracle(ctx):
    """§8(f) f4: the per-product recorder sees every product of an NS run (X, Y', Z' per
    k).  On C2 (30 iterations) each product's ijk task set equals the oracle's (same
    Y0, Z0, c; the oracle's own free run), its distance histogram equals the one counted
    from the oracle's triples, and the recorded counts equal spamm_ns_sqrt's stats."""
    c = si.CONFIGS["C2"]
    kind, payload = si.make_input(c)
    S, So = build_pair(ctx, kind, payload, c.b, c.n)
    cs = O.power_scale(So)
    nb = c.n // c.b
    sink = sp().VolumeSink(3 * c.iters, nbins=nb, ikj_cap=400000)
    sp().spamm_ctx_set_volume_sink(ctx, sink)
    try:
        r = sp().spamm_ns_sqrt(ctx, S, c.tau, c.iters, scale=cs)
    finally:
        sp().spamm_ctx_set_volume_sink(ctx, None)
    assert sink.nprod == 3 * c.iters and sink.complete()
    assert list(sink.ntasks) == [p["tasks"] for k in r["stats"] for p in k]
    Y, Z = O.ns_y0(So, cs), O.OMat.identity(c.n, c.b)
    for k in range(c.iters):
        Y, Z, _, _, _, tasks = O.ns_step(Y, Z, c.tau, want_tasks=True)
        for q in range(3):
            g = sink.tasks(3 * k + q)
            assert P.triples(g) == P.triples(tasks[q]), (k, q)
            d = np.max(np.abs(np.stack([g[:, 0] - g[:, 2], g[:, 0] - g[:, 1], g[:, 2] - g[:, 1]])), axis=0)
            assert np.array_equal(sink.hist[3 * k + q], np.bincount(np.minimum(d, nb - 1), minlength=nb))


def test_async_host_io_equals_sync(ctx):
    """The C ABI's asynchronous host I/O (upload on the library's upload stream, export on
    its copy stream) gives exactly the synchronous calls' results: a staged block list and
    a staged dense input build the same quadtrees, spamm_export_blocks_async writes the same
    blocks as spamm_export_blocks, and a third outstanding upload invalidates the first."""
    c = si.CONFIGS["C3"]
    _, (bi, bj, blocks) = si.make_input(c, n=4096)
    hb = [torch.from_numpy(x).pin_memory() for x in (bi, bj, blocks)]
    A = sp().spamm_build_tree_blocks(ctx, 4096, 64, *hb)
    A2 = sp().spamm_build_tree_staged(ctx, 4096, 64, sp().spamm_stage_blocks(ctx, 64, *hb))
    s = si.kms(1024, 0.8)
    D = sp().spamm_build_tree(ctx, s, 32)
    D2 = sp().spamm_build_tree_staged(ctx, 1024, 32, sp().spamm_stage_dense(ctx, torch.from_numpy(s).pin_memory()))
    for M, M2 in ((A, A2), (D, D2)):
        g1, g2 = sp().spamm_export_blocks(ctx, M), sp().spamm_export_blocks(ctx, M2)
        for x, y in zip(g1, g2):
            assert np.array_equal(x, y)
        L = (M.n // M.b).bit_length() - 1
        assert np.array_equal(sp().spamm_level_norms2(ctx, M, L), sp().spamm_level_norms2(ctx, M2, L))
        k = M.nblocks
        out = (torch.empty(k, dtype=torch.int32).pin_memory(), torch.empty(k, dtype=torch.int32).pin_memory(),
               torch.empty((k, M.b, M.b), dtype=torch.float64).pin_memory())
        assert sp().spamm_export_blocks_async(ctx, M, out) == k
        sp().spamm_copies_wait(ctx)
        for x, y in zip(g1, out):
            assert np.array_equal(x, y.numpy())
    h1 = sp().spamm_stage_blocks(ctx, 64, *hb)
    sp().spamm_stage_blocks(ctx, 64, *hb)
    sp().spamm_stage_blocks(ctx, 64, *hb)          # SPAMM_ISLOTS = 2: h1's slot is refilled
    with pytest.raises(sp().SpammError) as e:
        sp().spamm_build_tree_staged(ctx, 4096, 64, h1)
    assert e.value.code == 1


@pytest.mark.parametrize("case", ["C1", "b16_holes", "b32_reg"])
def test_power_cluster_bitwise(ctx, case):
    """Tiny s (C1: n = 256): the whole power iteration runs on one thread-block cluster
    with s resident in shared memory (power.cu k_power_cluster).  Its arithmetic is the
    launch loop's (register SpMV, k_normalize, k_dot), so c is bitwise the same with
    SPAMM_POWER_CLUSTER=0/1, and matches the oracle's power iteration (reading L12).
    Cases: the C1 input; n = 256 b = 16 with absent off-diagonal blocks and an empty
    block-row tail; n = 512 b = 32 on the register SpMV (SPAMM_SPMV_BLK=0, E = 4 lanes)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "import paper_1508_05856_b200 as sp, spamm_inputs as si, torch\n"
            "from test_gpu_parity import decaying\n"
            "ctx = sp.spamm_ctx_create(0); case = %r\n"
            "if case == 'C1':\n"
            "    c = si.CONFIGS['C1']; kind, p = si.make_input(c); n, b = c.n, c.b\n"
            "    m = p if kind == 'dense' else None\n"
            "    S = (sp.spamm_build_tree(ctx, torch.from_numpy(p).cuda(), b) if kind == 'dense' else\n"
            "         sp.spamm_build_tree_blocks(ctx, n, b, *(torch.from_numpy(x).cuda() for x in p)))\n"
            "else:\n"
            "    n, b = (256, 16) if case == 'b16_holes' else (512, 32)\n"
            "    m = np.abs(decaying(n, 0.02, 5)); m = m + m.T\n"
            "    if case == 'b16_holes':\n"
            "        r = np.random.default_rng(4)\n"
            "        for I in range(n // b):\n"
            "            for J in range(I + 1, n // b):\n"
            "                if r.random() < 0.4: m[I*b:(I+1)*b, J*b:(J+1)*b] = 0; m[J*b:(J+1)*b, I*b:(I+1)*b] = 0\n"
            "        m[n - b:, :] = 0; m[:, n - b:] = 0\n"
            "    S = sp.spamm_build_tree(ctx, torch.from_numpy(m).cuda(), b)\n"
            "print(repr(sp.spamm_power_scale(ctx, S, 100)))\n")
    out = []
    for mode in ("1", "0"):
        env = {**os.environ, "SPAMM_POWER_CLUSTER": mode}
        if case == "b32_reg":
            env["SPAMM_SPMV_BLK"] = "0"
        p = subprocess.run([sys.executable, "-c", code % (root, os.path.join(root, "tests"), case)],
                           capture_output=True, text=True, timeout=600, env=env)
        assert p.returncode == 0, p.stderr[-2000:]
        out.append(p.stdout.strip().splitlines()[-1])
    assert out[0] == out[1], out
    if case != "C1":
        n, b = (256, 16) if case == "b16_holes" else (512, 32)
        m = np.abs(decaying(n, 0.02, 5))
        m = m + m.T
        if case == "b16_holes":
            r = np.random.default_rng(4)
            for I in range(n // b):
                for J in range(I + 1, n // b):
                    if r.random() < 0.4:
                        m[I * b:(I + 1) * b, J * b:(J + 1) * b] = 0
                        m[J * b:(J + 1) * b, I * b:(I + 1) * b] = 0
            m[n - b:, :] = 0
            m[:, n - b:] = 0
        assert float(out[0]) == pytest.approx(O.power_scale(O.OMat.from_dense(m, b), 100), rel=1e-12)
