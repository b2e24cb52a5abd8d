"""CPU checks of the parity-comparison mechanics (tests/_parity.py), SURVEY.md §8(c):
the flip window and the flip correction, on a constructed case where two oracle runs
differ by exactly the at-threshold triples (no GPU involved)."""
import numpy as np

import _parity as P
import oracle as O


def test_flip_correction_reconstructs_the_other_side():
    # ones(32), b = 16: all 8 leaf triples sit exactly at T for tau = 1/4 (P:205 tie);
    # one ulp above, all are culled.  Treat the culled run as "the GPU".
    A = O.OMat.from_dense(np.ones((32, 32)), 16)
    Ck, tk = O.multiply(A, A, 0.25, want_tasks=True)
    Cc, tc = O.multiply(A, A, np.nextafter(0.25, 1.0), want_tasks=True)
    sk, sc = P.triples(tk), P.triples(tc)
    assert len(sk) == 8 and len(sc) == 0
    # every flipped triple is inside the window (|p - T| = 0 relative to tau = 1/4)
    assert P.outside_window(sk ^ sc, A, A, 0.25) == []
    # flip-correcting the kept run by the triples only it has gives the culled run
    corr = P.flip_correct(P.oracle_blocks(Ck), A, A, only_gpu=sc - sk, only_oracle=sk - sc)
    assert P.rel_union(P.oracle_blocks(Cc), corr) == 0.0
    for blk in corr.values():
        assert np.all(blk == 0.0)


def test_window_rejects_a_real_flip():
    # partial-cull fixture: the two-off-diagonal triples have n2 product 1/4096 < T,
    # far outside the window, so claiming them as flips must fail
    Pm = np.ones((16, 16)) / 16
    A = O.OMat.from_dense(np.block([[Pm, Pm / 8], [Pm / 8, Pm]]), 16)
    _, t = O.multiply(A, A, 1 / 32, want_tasks=True)
    s = P.triples(t)
    assert len(s) == 6
    culled = {(0, 1, 0), (1, 0, 1)}
    assert not (culled & s)
    assert sorted(P.outside_window(culled, A, A, 1 / 32)) == sorted(culled)


def test_rel_union_counts_one_sided_blocks():
    o = {(0, 0): np.ones((2, 2))}
    g = {(0, 0): np.ones((2, 2)), (1, 1): np.full((2, 2), 0.5)}
    assert P.rel_union(g, o) == np.sqrt(4 * 0.25) / 2.0
