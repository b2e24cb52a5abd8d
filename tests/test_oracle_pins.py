"""Pins of the CPU oracle against what PAPER.md and mathematics fix (CPU only).

Each test names the passage it pins.  None of these re-types the oracle's
formula: expected values come from closed forms, brute force, an independent
library routine (numpy matmul / eigh), constructed exact-binary cases, or the
paper's inequalities.
"""
import math
import os

import numpy as np
import pytest

import oracle as O
import spamm_inputs as si

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rng(seed):
    return np.random.default_rng(seed)


def decaying(n, rate, seed, sym=False, sign=True):
    """Test-local random matrix with exponential off-diagonal decay (and some
    exactly-zero far blocks through underflow-free hard zeroing)."""
    r = _rng(seed)
    i = np.arange(n)
    d = np.abs(i[:, None] - i[None, :])
    m = np.exp(-rate * d) * (r.standard_normal((n, n)) if sign else r.random((n, n)))
    m[d > n // 2] = 0.0
    if sym:
        m = 0.5 * (m + m.T)
    return m


def block_norms(m, b):
    nb = m.shape[0] // b
    return np.sqrt(np.einsum("ibjc,ibjc->ij", m.reshape(nb, b, nb, b), m.reshape(nb, b, nb, b)))


def flat_tasks(a, bm, b, tau):
    """Brute force over all nb^3 leaf triples with the flat test
    ||A_ik|| ||B_kj|| >= tau ||A|| ||B|| (present blocks only).  Returns the task set
    and the set of triples within 1e-12 relative of the threshold (ambiguous)."""
    na, nbm = block_norms(a, b), block_norms(bm, b)
    thr = tau * np.linalg.norm(a) * np.linalg.norm(bm)
    prod = na[:, :, None] * nbm[None, :, :]            # [i,k,j]
    present = (na[:, :, None] > 0) & (nbm[None, :, :] > 0)
    keep = present & (prod >= thr)
    amb = present & (np.abs(prod - thr) <= 1e-12 * max(thr, 1e-300))
    return ({tuple(x) for x in np.argwhere(keep)}, {tuple(x) for x in np.argwhere(amb)})


# --------------------------------------------------------------- quadtree
@pytest.mark.parametrize("n,b", [(64, 16), (128, 16), (256, 32), (64, 64)])
def test_norms_root_and_recursion(n, b):
    """root = dense Frobenius; parent^2 = sum children^2."""
    m = decaying(n, 0.05, n + b)
    A = O.OMat.from_dense(m, b)
    assert abs(A.norm() - np.linalg.norm(m)) <= 1e-14 * np.linalg.norm(m)
    L = (n // b).bit_length() - 1
    leaf = A.level_norms(L)
    np.testing.assert_allclose(leaf, block_norms(m, b), rtol=1e-14, atol=0)
    for lev in range(L):
        p = A.level_norms(lev)
        c = A.level_norms(lev + 1) ** 2
        s = c[0::2, 0::2] + c[0::2, 1::2] + c[1::2, 0::2] + c[1::2, 1::2]
        np.testing.assert_allclose(p ** 2, s, rtol=1e-14, atol=0)


def test_roundtrip_and_blocks():
    m = decaying(128, 0.2, 3)
    m[:16, 32:48] = 0.0                       # an absent block
    A = O.OMat.from_dense(m, 16)
    assert np.array_equal(A.to_dense(), m)
    bi, bj = A.block_coords()
    present = block_norms(m, 16) > 0
    assert len(bi) == present.sum() and not present[0, 2]
    blocks = np.stack([m[i * 16:(i + 1) * 16, j * 16:(j + 1) * 16] for i, j in zip(bi, bj)])
    B = O.OMat.from_blocks(128, 16, bi, bj, blocks)
    assert np.array_equal(B.to_dense(), m)
    assert B.norm() == A.norm()


# ---------------------------------------------------------------- SpAMM
def test_tiebreak_strict_inequality_golden():
    """P:205 strict '<' at exact equality (tests/golden/tiebreak.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLD, "tiebreak.txt")) if not l.startswith("#")]
    A = O.OMat.from_dense(np.ones((32, 32)), 16)
    for tau_hex, nt, val in rows:
        C, t = O.multiply(A, A, float.fromhex(tau_hex), want_tasks=True)
        assert len(t) == int(nt)
        assert np.all(C.to_dense() == float(val))


def test_partial_cull_golden():
    """Eq. newspamm + Proposition on an exact-binary constructed case."""
    lines = [l for l in open(os.path.join(GOLD, "partial_cull.txt")) if not l.startswith("#")]
    expect = {tuple(int(x) for x in l.split()) for l in lines if l.strip()}
    P = np.ones((16, 16)) / 16
    eps = 1.0 / 8
    A = np.block([[P, eps * P], [eps * P, P]])
    Ao = O.OMat.from_dense(A, 16)
    assert Ao.norm() ** 2 == 2.03125
    C, t = O.multiply(Ao, Ao, 1.0 / 32, want_tasks=True)
    assert {tuple(x) for x in t} == expect
    Cd = C.to_dense()
    assert np.array_equal(Cd, np.block([[P, P / 4], [P / 4, P]]))
    D = Cd - A @ A
    assert np.array_equal(D, np.block([[-eps ** 2 * P, 0 * P], [0 * P, -eps ** 2 * P]]))
    assert np.linalg.norm(D) == pytest.approx(math.sqrt(2) / 64, rel=1e-15)


@pytest.mark.parametrize("n,b,seed", [(64, 16, 1), (128, 16, 2), (256, 32, 3), (256, 16, 4),
                                      (128, 64, 5)])
def test_tau0_is_dense_gemm(n, b, seed):
    """as tau -> 0 SpAMM reverts to the (recursive) GEMM."""
    a = decaying(n, 0.03, seed)
    bm = decaying(n, 0.05, seed + 100)
    a[0:b, 2 * b:3 * b] = 0.0                      # absent blocks never form tasks
    C, t = O.multiply(O.OMat.from_dense(a, b), O.OMat.from_dense(bm, b), 0.0, want_tasks=True)
    ref = a @ bm
    assert np.linalg.norm(C.to_dense() - ref) <= 1e-13 * np.linalg.norm(ref)
    pa, pb = block_norms(a, b) > 0, block_norms(bm, b) > 0
    assert len(t) == int(np.einsum("ik,kj->", pa.astype(int), pb.astype(int)))


@pytest.mark.parametrize("tau", [1e-1, 1e-2, 1e-3, 1e-4, 1e-6])
@pytest.mark.parametrize("seed", [11, 12, 13])
def test_error_bounds(tau, seed):
    """Proposition: |Delta_ij| <= n tau_ab and ||Delta|| <= n^2 tau_ab;
    plus the derived culled-mass bound ||Delta|| <= ||[sum_culled ||A_ik|| ||B_kj||]_ij||."""
    n, b = 128, 16
    a = decaying(n, 0.1, seed)
    bm = decaying(n, 0.15, seed + 50)
    C, t = O.multiply(O.OMat.from_dense(a, b), O.OMat.from_dense(bm, b), tau, want_tasks=True)
    D = C.to_dense() - a @ bm
    tab = tau * np.linalg.norm(a) * np.linalg.norm(bm)
    assert np.max(np.abs(D)) <= n * tab
    assert np.linalg.norm(D) <= n * n * tab
    na, nbm = block_norms(a, b), block_norms(bm, b)
    full = np.einsum("ik,kj->ikj", na, nbm)
    kept = np.zeros_like(full, dtype=bool)
    kept[tuple(t.T)] = True
    culled_mass = np.where(kept, 0.0, full).sum(axis=1)
    assert np.linalg.norm(D) <= np.linalg.norm(culled_mass) * (1 + 1e-12) + 1e-300


@pytest.mark.parametrize("tau", [0.0, 1e-2, 1e-3, 1e-5, 1e-8])
@pytest.mark.parametrize("n,b", [(128, 16), (256, 16), (256, 32)])
def test_recursive_equals_flat_bruteforce(tau, n, b):
    """The recursive two-sided query (Eq. newspamm) returns exactly the flat leaf
    test set (monotone norms), modulo the 1e-12 threshold window."""
    a = decaying(n, 0.05, 7 + n)
    bm = decaying(n, 0.08, 9 + b)
    _, t = O.multiply(O.OMat.from_dense(a, b), O.OMat.from_dense(bm, b), tau, want_tasks=True)
    got = {tuple(x) for x in t}
    want, amb = flat_tasks(a, bm, b, tau)
    assert (got ^ want) <= amb


def test_special_cases():
    """S:139 / P:205: tau slightly > 1 culls everything (the root pair fails);
    tau = 1 keeps the root pair; a single-block A and B sharing k survive at tau=1."""
    a = decaying(64, 0.1, 21)
    A = O.OMat.from_dense(a, 16)
    C, t = O.multiply(A, A, np.nextafter(1.0, 2.0), want_tasks=True)
    assert len(t) == 0 and C.nblocks() == 0
    e = np.zeros((64, 64))
    e[16:32, 32:48] = _rng(5).standard_normal((16, 16))   # A = single block (1,2)
    f = np.zeros((64, 64))
    f[32:48, 0:16] = _rng(6).standard_normal((16, 16))    # B = single block (2,0)
    C, t = O.multiply(O.OMat.from_dense(e, 16), O.OMat.from_dense(f, 16), 1.0, want_tasks=True)
    assert [tuple(x) for x in t] == [(1, 2, 0)]
    ref = e @ f
    assert np.linalg.norm(C.to_dense() - ref) <= 1e-14 * np.linalg.norm(ref)


def test_identity_left_operand_rule():
    """I (x)_tau B keeps (i,i,j) iff ||I_ii|| ||B_ij|| >= tau ||I|| ||B||, i.e.
    b * n^2_B[i,j] >= tau^2 * n * ||B||^2 (closed form of the flat test)."""
    n, b, tau = 256, 16, 1e-3
    bm = decaying(n, 0.05, 31)
    I = O.OMat.identity(n, b)
    assert np.array_equal(I.to_dense(), np.eye(n))
    _, t = O.multiply(I, O.OMat.from_dense(bm, b), tau, want_tasks=True)
    nbm2 = block_norms(bm, b) ** 2
    lhs = b * nbm2
    rhs = tau ** 2 * n * np.linalg.norm(bm) ** 2
    want = {(i, i, j) for i, j in np.argwhere((lhs >= rhs) & (nbm2 > 0))}
    amb = {(i, i, j) for i, j in np.argwhere(np.abs(lhs - rhs) <= 1e-12 * rhs)}
    assert ({tuple(x) for x in t} ^ want) <= amb
    assert all(x[0] == x[1] for x in t)


def test_tau_monotone_work():
    """the surviving task set is nested, decreasing in tau."""
    a, bm = decaying(256, 0.05, 41), decaying(256, 0.05, 42)
    A, B = O.OMat.from_dense(a, 16), O.OMat.from_dense(bm, 16)
    prev = None
    for tau in [0.0, 1e-8, 1e-6, 1e-4, 1e-2, 1e-1]:
        _, t = O.multiply(A, B, tau, want_tasks=True)
        s = {tuple(x) for x in t}
        if prev is not None:
            assert s <= prev
        prev = s


def test_transpose_symmetry():
    """(A (x) B)^T = B^T (x) A^T (same task set modulo the window; values to rounding)."""
    n, b, tau = 256, 16, 1e-4
    a, bm = decaying(n, 0.05, 51), decaying(n, 0.07, 52)
    C, t = O.multiply(O.OMat.from_dense(a, b), O.OMat.from_dense(bm, b), tau, want_tasks=True)
    Ct, tt = O.multiply(O.OMat.from_dense(bm.T.copy(), b), O.OMat.from_dense(a.T.copy(), b),
                        tau, want_tasks=True)
    s1 = {(i, k, j) for i, k, j in t}
    s2 = {(j, k, i) for i, k, j in tt}
    _, amb = flat_tasks(a, bm, b, tau)
    assert (s1 ^ s2) <= amb
    np.testing.assert_allclose(Ct.to_dense().T, C.to_dense(), rtol=0,
                               atol=1e-14 * np.abs(C.to_dense()).max())


# ---------------------------------------------------------- Newton-Schulz
def _eig_pow(s, p):
    w, V = np.linalg.eigh(s)
    return (V * w ** p) @ V.T


def test_ns_identity_fixed_point():
    """Fixed point: s = I stays at Y = Z = I, t_k = 0."""
    S = O.OMat.from_dense(np.eye(64), 16)
    r = O.ns_sqrt(S, 1e-6, 5)
    assert np.abs(r["Y"].to_dense() - np.eye(64)).max() <= 1e-15
    assert np.abs(r["Z"].to_dense() - np.eye(64)).max() <= 1e-15
    assert np.all(np.abs(r["t"]) <= 1e-15)


def test_ns_scalar_4I():
    """s = 4I -> Y = 2I, Z = I/2."""
    S = O.OMat.from_dense(4 * np.eye(64), 16)
    r = O.ns_sqrt(S, 0.0, 8)
    assert r["c"] == pytest.approx(4.0, rel=1e-15)
    assert np.abs(r["Y"].to_dense() - 2 * np.eye(64)).max() <= 1e-15
    assert np.abs(r["Z"].to_dense() - 0.5 * np.eye(64)).max() <= 1e-15


def test_ns_diagonal_scalar_recursion():
    """Eq. cannonical with commuting diagonal iterates decouples into the scalar map
    x = z y, h = (3 - x)/2, y' = y h, z' = h z, at tau = 0: bitwise."""
    n, b = 64, 16
    lam = np.linspace(0.05, 1.0, n)[_rng(3).permutation(n)]
    S = O.OMat.from_dense(np.diag(lam), b)
    c = 1.0
    Y = O.ns_y0(S, c)
    Z = O.OMat.identity(n, b)
    y, z = lam / c, np.ones(n)
    for k in range(20):
        Y, Z, H, t, _ = O.ns_step(Y, Z, 0.0)
        x = z * y
        h = 0.5 * (3.0 - x)
        y, z = y * h, h * z
        assert np.array_equal(np.diag(Y.to_dense()), y), k
        assert np.array_equal(np.diag(Z.to_dense()), z), k
        assert np.array_equal(np.diag(H.to_dense()), h), k
        assert t == pytest.approx((n - x.sum()) / n, abs=1e-15)


@pytest.mark.parametrize("rho,n,b,iters", [(0.5, 256, 16, 25), (0.8, 256, 32, 30)])
def test_ns_kms_closed_forms(rho, n, b, iters):
    """KMS facts: s^{-1} is tridiagonal with diagonal (1+rho^2)/(1-rho^2) (corners
    1/(1-rho^2)) and off-diagonal -rho/(1-rho^2).  At tau = 0: Z.Z = s^{-1},
    Y.Y = s, YZ -> I, ZsZ -> I (BJ:5)."""
    s = si.kms(n, rho)
    S = O.OMat.from_dense(s, b)
    r = O.ns_sqrt(S, 0.0, iters)
    Y, Z = r["Y"].to_dense(), r["Z"].to_dense()
    inv = np.zeros((n, n))
    k = 1.0 / (1 - rho ** 2)
    inv[np.arange(n), np.arange(n)] = (1 + rho ** 2) * k
    inv[0, 0] = inv[-1, -1] = k
    inv[np.arange(n - 1), np.arange(1, n)] = -rho * k
    inv[np.arange(1, n), np.arange(n - 1)] = -rho * k
    assert np.linalg.norm(Z @ Z - inv) <= 1e-12 * np.linalg.norm(inv)
    assert np.linalg.norm(Y @ Y - s) <= 1e-12 * np.linalg.norm(s)
    assert np.linalg.norm(Y @ Z - np.eye(n)) / math.sqrt(n) <= 1e-13
    assert np.linalg.norm(Z @ s @ Z - np.eye(n)) / math.sqrt(n) <= 1e-12
    lo, hi = (1 - rho) / (1 + rho), (1 + rho) / (1 - rho)
    assert lo < r["c"] < hi


@pytest.mark.parametrize("seed", [1, 2])
def test_ns_eig_tiny(seed):
    """BJ:5: on tiny matrices s^{+-1/2} matches a brute-force eigendecomposition."""
    n, b = 128, 16
    g = _rng(seed).standard_normal((n, n)) * np.exp(-0.05 * np.abs(np.subtract.outer(
        np.arange(n), np.arange(n))))
    s = g @ g.T / n + 0.5 * np.eye(n)
    r = O.ns_sqrt(O.OMat.from_dense(s, b), 0.0, 40)
    for M, p in ((r["Y"], 0.5), (r["Z"], -0.5)):
        ref = _eig_pow(s, p)
        assert np.linalg.norm(M.to_dense() - ref) <= 1e-12 * np.linalg.norm(ref)


def test_ns_mu_shift():
    """Reading L13: Y0 = (s/c + mu I)/(1+mu) gives (s + c mu I)^{+-1/2} at tau = 0."""
    n, b, mu = 128, 16, 1e-2
    s = si.kms(n, 0.7)
    S = O.OMat.from_dense(s, b)
    r = O.ns_sqrt(S, 0.0, 40, mu=mu)
    sm = s + r["c"] * mu * np.eye(n)
    assert np.linalg.norm(r["Y"].to_dense() - _eig_pow(sm, 0.5)) <= 1e-12 * np.linalg.norm(sm)
    ref = _eig_pow(sm, -0.5)
    assert np.linalg.norm(r["Z"].to_dense() - ref) <= 1e-12 * np.linalg.norm(ref)


def test_ns_h_map_and_trace():
    """H = 1/2 (3I - X) (alpha = 1), X = Z (x)_tau Y, t = (n - tr X)/n."""
    n, b, tau = 256, 16, 1e-5
    s = si.kms(n, 0.6)
    S = O.OMat.from_dense(s, b)
    Y = O.ns_y0(S, O.power_scale(S))
    Z = O.OMat.identity(n, b)
    for _ in range(3):
        X = O.multiply(Z, Y, tau)
        Yn, Zn, H, t, _ = O.ns_step(Y, Z, tau)
        Xd = X.to_dense()
        assert np.array_equal(H.to_dense(), 0.5 * (3 * np.eye(n) - Xd))
        assert t == pytest.approx((n - np.trace(Xd)) / n, abs=1e-14)
        # Y' = Y (x) H and Z' = H (x) Z with the same H
        assert np.array_equal(Yn.to_dense(), O.multiply(Y, H, tau).to_dense())
        assert np.array_equal(Zn.to_dense(), O.multiply(H, Z, tau).to_dense())
        Y, Z = Yn, Zn


def test_ns_tau_accuracy_and_lensing_c1():
    """C1 (BJ:7) at tau = 1e-6: SpAMM-level accuracy ~1e-5 vs eigh, and after
    convergence the Y (x) H / H (x) Z task counts collapse to nnzb(Y), nnzb(Z)
    ("copy in place")."""
    cfg = si.CONFIGS["C1"]
    s = si.kms(cfg.n, cfg.rho)
    S = O.OMat.from_dense(s, cfg.b)
    r = O.ns_sqrt(S, cfg.tau, cfg.iters)
    for M, p in ((r["Y"], 0.5), (r["Z"], -0.5)):
        ref = _eig_pow(s, p)
        assert np.linalg.norm(M.to_dense() - ref) <= 1e-4 * np.linalg.norm(ref)
    assert abs(r["t"][-1]) < 1e-6
    cnt = r["counts"][-1]
    assert cnt[1] == r["Y"].nblocks() and cnt[2] == r["Z"].nblocks()


def test_power_scale():
    """Reading L12: Rayleigh quotient of K=100 power steps is <= lambda_max and
    close to it for a well-separated top eigenvalue."""
    s = si.kms(256, 0.9)
    S = O.OMat.from_dense(s, 16)
    c = O.power_scale(S, 100)
    lmax = np.linalg.eigvalsh(s)[-1]
    assert c <= lmax * (1 + 1e-15)
    assert c >= 0.99 * lmax


@pytest.mark.parametrize("K", [0, 1, 3, 10])
def test_power_scale_rayleigh_closed_form(K):
    """Reading L12: c = v_K^T s v_K after K normalised power steps from
    v_0 = 1/sqrt(n) 1.  For s = diag(2 I_{n/2}, I_{n/2}), v_K is proportional to
    [2^K 1, 1], so c = (2^(2K+1) + 1)/(2^(2K) + 1) exactly; the norm ||s v_K||
    (a plausible mistake) would give sqrt((2^(2K+2) + 1)/(2^(2K) + 1)) instead."""
    n, b = 64, 16
    s = np.diag(np.r_[np.full(n // 2, 2.0), np.ones(n // 2)])
    c = O.power_scale(O.OMat.from_dense(s, b), K)
    exact = (2.0 ** (2 * K + 1) + 1) / (2.0 ** (2 * K) + 1)
    wrong = np.sqrt((2.0 ** (2 * K + 2) + 1) / (2.0 ** (2 * K) + 1))
    assert c == pytest.approx(exact, rel=1e-14)
    assert wrong != pytest.approx(exact, rel=1e-10)   # the pin tells them apart


def test_ns_y0_mu_fills_absent_diagonal_blocks():
    """Op 1 (reading L13): Y0 = (s/c + mu I)/(1+mu) everywhere, including diagonal blocks
    that s does not store (there Y0_ii = mu/(1+mu) I), against numpy on the dense s."""
    n, b, c, mu = 128, 16, 3.0, 1e-2
    s = np.abs(_rng(11).standard_normal((n, n)))
    s = s + s.T
    for I in (2, 5):                   # diagonal blocks absent from s
        s[I * b:(I + 1) * b, I * b:(I + 1) * b] = 0.0
    s[0:b, 3 * b:4 * b] = s[3 * b:4 * b, 0:b] = 0.0   # and an off-diagonal pair
    S = O.OMat.from_dense(s, b)
    assert S.block(2, 2) is None and S.block(5, 5) is None
    Y0 = O.ns_y0(S, c, mu)
    ref = (s / c + mu * np.eye(n)) / (1 + mu)
    assert np.array_equal(Y0.to_dense(), ref)
    assert np.array_equal(Y0.block(2, 2), mu / (1 + mu) * np.eye(b))
    assert Y0.block(0, 3) is None       # only the diagonal is filled
    assert Y0.nblocks() == S.nblocks() + 2
    # mu = 0: the plain s/c, absent blocks stay absent
    assert O.ns_y0(S, c).block(2, 2) is None


# ------------------------------------------- scaled / stabilised map (§8(f) f1)
def test_scaled_map_sigmoids_paper_values():
    """alpha(t) = 1 + 1.85/(1 + e^{-50(t-.35)}), eps(t) = .1/(1 + e^{-75(t-.30)}):
    midpoints alpha(.35) = 1.925, eps(.30) = .05; saturation alpha -> 2.85, eps -> .1 for
    t -> 1; both damped to (1, 0) as t -> 0."""
    assert O.alpha(0.35) == pytest.approx(1.925, rel=1e-15)
    assert O.eps(0.30) == pytest.approx(0.05, rel=1e-15)
    assert O.alpha(1.0) == pytest.approx(2.85, rel=1e-12)
    assert O.eps(1.0) == pytest.approx(0.1, rel=1e-15)
    assert 1.0 < O.alpha(0.0) < 1.0 + 1e-7 and 0.0 < O.eps(0.0) < 1e-10
    ts = np.linspace(0, 1, 101)
    assert np.all(np.diff([O.alpha(t) for t in ts]) >= 0)
    assert np.all(np.diff([O.eps(t) for t in ts]) >= 0)
    ts = np.linspace(0.1, 0.6, 51)          # strictly increasing away from saturation
    assert np.all(np.diff([O.alpha(t) for t in ts]) > 0)
    assert np.all(np.diff([O.eps(t) for t in ts]) > 0)


def test_scaled_map_h_of_x():
    """H = sqrt(alpha)/2 (3I - alpha((1-2eps) X + eps I)) with alpha(t_k), eps(t_k): for a
    diagonal X the map is the scalar logistic h_alpha of the shifted-scaled eigenvalue,
    whose fixed-point product h^2 x equals the standard NS map g(u) = u(3-u)^2/4 at
    u = alpha x~ scaled by x / x~."""
    n, b = 64, 16
    lam = np.linspace(0.02, 1.0, n)
    S = O.OMat.from_dense(np.diag(lam), b)
    Y, Z = O.ns_y0(S, 1.0), O.OMat.identity(n, b)
    Yn, Zn, H, t, _ = O.ns_step(Y, Z, 0.0, scaled=True)
    a, e = O.alpha(t), O.eps(t)
    x = lam
    xt = (1 - 2 * e) * x + e
    u = a * xt
    h = np.diag(H.to_dense())
    assert a > 2.5 and e > 0.09      # t_0 ~ .49: strongly scaled, stabilised
    # h^2 x~ = g(u): the NS logistic in the scaled variable u = alpha x~
    np.testing.assert_allclose(h * h * xt, u * (3 - u) ** 2 / 4, rtol=1e-14)
    assert t == pytest.approx(1 - lam.mean(), abs=1e-15)
    assert np.count_nonzero(H.to_dense() - np.diag(h)) == 0


def test_scaled_converges_to_eig_and_accelerates():
    """At tau = 0 the scaled/stabilised iteration still converges to s^{+-1/2}
    (eigendecomposition; the sigmoids leave alpha - 1 ~ 5e-8, eps ~ 2e-11 at t = 0, so
    the fixed point is shifted by O(eps)), and reaches t_k < 1e-10 in fewer steps than
    the plain map on an ill-conditioned s (the purpose of the scaling)."""
    n, b = 128, 16
    g = _rng(5).standard_normal((n, n)) * np.exp(-0.05 * np.abs(np.subtract.outer(np.arange(n), np.arange(n))))
    s = g @ g.T / n
    w, V = np.linalg.eigh(s)
    w = np.geomspace(1e-4, 1.0, n)                    # kappa = 1e4
    s = (V * w) @ V.T
    s = 0.5 * (s + s.T)
    S = O.OMat.from_dense(s, b)
    plain = O.ns_sqrt(S, 0.0, 60, scale=1.0, t_stop=1e-10)
    scaled = O.ns_sqrt(S, 0.0, 60, scale=1.0, t_stop=1e-10, scaled=True)
    assert scaled["iters"] < plain["iters"] <= 60
    for M, p in ((scaled["Y"], 0.5), (scaled["Z"], -0.5)):
        ref = _eig_pow(s, p)
        assert np.linalg.norm(M.to_dense() - ref) <= 1e-9 * np.linalg.norm(ref)


def test_t_stop_prefix():
    """t_stop ends the run at the first k with |t_k| <= t_stop; the history
    is the prefix of the fixed-count run."""
    cfg = si.CONFIGS["C1"]
    S = O.OMat.from_dense(si.kms(cfg.n, cfg.rho), cfg.b)
    full = O.ns_sqrt(S, cfg.tau, cfg.iters, scale=3.0)
    stop = O.ns_sqrt(S, cfg.tau, cfg.iters, scale=3.0, t_stop=1e-6)
    k = stop["iters"]
    assert 0 < k < cfg.iters
    assert np.array_equal(stop["t"], full["t"][:k])
    assert abs(stop["t"][-1]) <= 1e-6 and np.all(np.abs(full["t"][:k - 1]) > 1e-6)


# ------------------------------------------- single channel (§8(f) f2)
def test_transpose_and_multiply_t():
    """A^T (x)_tau B: tau = 0 equals numpy A.T @ B; the task set is the brute-force leaf
    test on the transposed norms ||A_ki|| ||B_kj|| >= tau ||A|| ||B||; the
    transpose is an involution that carries the norms over."""
    n, b = 256, 16
    r = _rng(11)
    i = np.arange(n)
    a = np.exp(-0.05 * np.abs(i[:, None] - i[None, :])) * r.standard_normal((n, n))
    c = np.exp(-0.03 * np.abs(i[:, None] - i[None, :])) * r.standard_normal((n, n))
    a[:b, 3 * b:4 * b] = 0.0
    A, B = O.OMat.from_dense(a, b), O.OMat.from_dense(c, b)
    At = O.transpose(A)
    assert np.array_equal(At.to_dense(), a.T)
    assert np.array_equal(O.transpose(At).to_dense(), a)
    assert At.norm() == A.norm()
    C0 = O.multiply(A, B, 0.0, trans_a=True)
    assert np.linalg.norm(C0.to_dense() - a.T @ c) <= 1e-13 * np.linalg.norm(a.T @ c)
    for tau in (1e-4, 1e-2):
        Ct, tasks = O.multiply(A, B, tau, want_tasks=True, trans_a=True)
        na, nb_ = A.leaf_norms(), B.leaf_norms()          # na[k, i] = ||A_ki||
        thr = tau * A.norm() * B.norm()
        prod = na.T[:, :, None] * nb_[None, :, :]          # [i, k, j]
        brute = {tuple(x) for x in np.argwhere((na.T[:, :, None] > 0) & (nb_[None] > 0) & (prod >= thr))}
        got = {tuple(x) for x in tasks}
        amb = {tuple(x) for x in np.argwhere(np.abs(prod - thr) <= 1e-12 * thr)}
        assert (got ^ brute) <= amb


def test_single_channel_tau0_matches_eig_and_dual():
    """P:398-402 at tau = 0: Z -> s^{-1/2}, Y = s Z -> s^{1/2}; the single and dual
    channels are the same iteration in exact arithmetic (z_k commutes with s)."""
    n, b = 128, 16
    g = _rng(4).standard_normal((n, n)) * np.exp(-0.05 * np.abs(np.subtract.outer(np.arange(n), np.arange(n))))
    s = g @ g.T / n + 0.5 * np.eye(n)
    S = O.OMat.from_dense(s, b)
    r1 = O.ns_sqrt_single(S, 0.0, 40)
    r2 = O.ns_sqrt(S, 0.0, 40)
    for M, p in ((r1["Y"], 0.5), (r1["Z"], -0.5)):
        ref = _eig_pow(s, p)
        assert np.linalg.norm(M.to_dense() - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.norm(r1["Z"].to_dense() - r2["Z"].to_dense()) <= 1e-12 * np.linalg.norm(r2["Z"].to_dense())
    assert abs(r1["t"][-1]) < 1e-14


def test_single_channel_diagonal_scalar_map():
    """Diagonal s: the single channel decouples into z' = z h(x), x' = z'^2 lambda/c
    (P:398-402 with commuting scalars); at tau = 0 the iterates match to 1 ulp-level."""
    n, b = 64, 16
    lam = np.linspace(0.1, 1.0, n)
    S = O.OMat.from_dense(np.diag(lam), b)
    r = O.ns_sqrt_single(S, 0.0, 12, scale=1.0)
    z, x = np.ones(n), lam.copy()
    for k in range(12):
        assert r["t"][k] == pytest.approx((n - x.sum()) / n, abs=1e-15)
        h = 0.5 * (3.0 - x)
        z = z * h
        x = z * (lam * z)
    np.testing.assert_allclose(np.diag(r["Z"].to_dense()), z, rtol=1e-15)
    assert r["counts"].shape == (12, 3)


# ------------------------------------- regularised product representation (§8(f) f3)
def _ill_conditioned(n, kappa, seed):
    g = _rng(seed).standard_normal((n, n)) * np.exp(-0.05 * np.abs(np.subtract.outer(np.arange(n), np.arange(n))))
    _, V = np.linalg.eigh(g @ g.T)
    w = np.geomspace(1.0 / kappa, 1.0, n)
    s = (V * w) @ V.T
    return 0.5 * (s + s.T)


def test_regularized_factor_tau0_inverse_factor():
    """P:748-776 at tau0 = tau1 = 0: G^T (s + c mu_m I) G = I; one slice is the inverse square
    root (s + c mu_0 I)^{-1/2} of the shifted matrix (the 'MAYEBOO' preconditioner)."""
    n, b = 128, 16
    s = _ill_conditioned(n, 1e6, 21)
    S = O.OMat.from_dense(s, b)
    mus = [1e-1, 1e-2, 1e-3]
    r = O.regularized_factor(S, 0.0, 0.0, mus, 60, t_stop=1e-13)
    G, c = r["G"].to_dense(), r["c"]
    sm = s + c * mus[-1] * np.eye(n)
    assert np.linalg.norm(G.T @ sm @ G - np.eye(n)) / np.sqrt(n) <= 1e-11
    r1 = O.regularized_factor(S, 0.0, 0.0, mus[:1], 60, t_stop=1e-13)
    ref = _eig_pow(s + r1["c"] * mus[0] * np.eye(n), -0.5)
    assert np.linalg.norm(r1["G"].to_dense() - ref) <= 1e-11 * np.linalg.norm(ref)


def test_regularized_slices_effective_by_one_order():
    """Each residual R_i = F^T (s/c + mu_i I) F is 'effective by one order': its
    condition number is ~ mu_{i-1}/mu_i = 10, whatever kappa(s) (here 1e6), so every slice
    solves a well-conditioned problem; checked at tau = 0 with the exact eigenvalues."""
    n, b = 128, 16
    s = _ill_conditioned(n, 1e6, 22)
    S = O.OMat.from_dense(s, b)
    c = O.power_scale(S)
    mus = [1e-1, 1e-2, 1e-3, 1e-4]
    for i in range(1, len(mus)):
        F = O.regularized_factor(S, 0.0, 0.0, mus[:i], 60, t_stop=1e-13, scale=c)["G"].to_dense() * np.sqrt(c)
        R = F.T @ (s / c + mus[i] * np.eye(n)) @ F
        w = np.linalg.eigvalsh(0.5 * (R + R.T))
        assert w.max() / w.min() <= 1.05 * mus[i - 1] / mus[i]
    ws = np.linalg.eigvalsh(s / c + mus[-1] * np.eye(n))
    assert ws.max() / ws.min() > 5e3           # the unsliced problem is far worse conditioned
