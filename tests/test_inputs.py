"""Input-generator checks (spamm_inputs): Hilbert curve brute force, KMS closed
form, Gaussian overlap symmetry and the lossless block-drop invariant."""
import math

import numpy as np
import pytest

import spamm_inputs as si


@pytest.mark.parametrize("bits", [1, 2, 3])
def test_hilbert_bruteforce(bits):
    """Skilling transpose Hilbert key on a 2^bits cube: a bijection onto
    [0, 8^bits) whose consecutive cells are face neighbours."""
    g = 1 << bits
    cells = np.array([(x, y, z) for x in range(g) for y in range(g) for z in range(g)])
    k = si.hilbert_keys(cells, bits)
    assert sorted(k.tolist()) == list(range(g ** 3))
    path = cells[np.argsort(k)]
    assert np.all(np.abs(np.diff(path, axis=0)).sum(axis=1) == 1)
    assert tuple(path[0]) == (0, 0, 0)


def test_kms_entries():
    s = si.kms(64, 0.9)
    assert np.array_equal(s, s.T)
    assert s[3, 10] == 0.9 ** 7
    assert np.all(np.diag(s) == 1.0)


def test_splitmix64_reference_value():
    # splitmix64 with seed 0: first output is the published test value of the algorithm
    assert int(si.splitmix64(0, 1)[0]) == 0xE220A8397B1DCDAF


def test_points_unit_density():
    n = 4096
    box = n ** (1 / 3)
    p = si.uniform_points(n, 7, box)
    assert p.shape == (n, 3) and p.min() >= 0 and p.max() < box
    assert abs(p.mean() - box / 2) < 0.05 * box


def test_gaussian_blocks_symmetric_and_lossless():
    n, b, sigma, shift, tau = 2048, 64, 0.8, 1e-3, 1e-7
    box = n ** (1 / 3)
    pts = si.uniform_points(n, 123, box)
    pts = pts[si.hilbert_order(pts, box)]
    delta = 1e-2 * tau * math.sqrt(n)
    bi, bj, blocks = si.gaussian_blocks(pts, b, sigma, shift, delta)
    dense = si.gaussian_dense(pts, sigma, shift)
    kept = {(i, j): k for k, (i, j) in enumerate(zip(bi, bj))}
    nb = n // b
    for I in range(nb):
        for J in range(nb):
            blk = dense[I * b:(I + 1) * b, J * b:(J + 1) * b]
            f = np.linalg.norm(blk)
            if (I, J) in kept:
                np.testing.assert_allclose(blocks[kept[(I, J)]], blk, rtol=1e-12, atol=0)
                assert (J, I) in kept
                assert np.array_equal(blocks[kept[(I, J)]], blocks[kept[(J, I)]].T)
                assert f >= delta * (1 - 1e-12)
            else:
                assert f < delta * (1 + 1e-12)
    # drop tolerance is below tau * ||s|| (lossless: dropped blocks can never survive)
    assert delta <= tau * np.linalg.norm(dense)


def test_gaussian_row_shards_equal_full_generation():
    """A rank's row shard (rows=(r0, r1)) is bitwise the matching slice of the full list."""
    cfg = si.Config("t", "gauss", 2048, 64, 1e-7, 30, sigma=0.8, shift=1e-3, seed=150805858, tau_min=1e-7)
    _, (bi, bj, blocks) = si.make_input(cfg)
    nb = 2048 // 64
    got = []
    for r0, r1 in [(0, 7), (7, 7), (7, 20), (20, nb)]:
        _, (si_, sj_, sb_) = si.make_input(cfg, rows=(r0, r1))
        assert np.all((si_ >= r0) & (si_ < r1))
        got.append((si_, sj_, sb_))
    assert np.array_equal(np.concatenate([g[0] for g in got]), bi)
    assert np.array_equal(np.concatenate([g[1] for g in got]), bj)
    assert np.array_equal(np.concatenate([g[2] for g in got]), blocks)
