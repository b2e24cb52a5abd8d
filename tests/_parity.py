"""Shared GPU-vs-oracle comparison helpers (SURVEY.md §8(c) parity protocol).

* Task sets: identical except triples whose norm product lies within 1e-12 relative
  of the threshold T = tau ||A|| ||B|| (the window, north_star BJ:5).  The window is
  evaluated only on the triples that differ, with the oracle's leaf norms.
* Values: relative Frobenius error over the UNION of both sides' stored blocks (a
  block present on one side only counts in full), after the flip correction of
  §8(c): for a triple only the GPU kept, A_ik B_kj is added to the oracle's C_ij;
  for one only the oracle kept, it is subtracted.
"""
from __future__ import annotations

import math

import numpy as np

WINDOW = 1e-12


def gpu_blocks(sp, ctx, M) -> dict:
    """{(I, J): block} of a GPU matrix (local rows on a row-partitioned context)."""
    bi, bj, blk = sp.spamm_export_blocks(ctx, M)
    return {(int(i), int(j)): blk[t] for t, (i, j) in enumerate(zip(bi, bj))}


def oracle_blocks(Mo) -> dict:
    bi, bj = Mo.block_coords()
    return {(int(i), int(j)): Mo.block(int(i), int(j)) for i, j in zip(bi, bj)}


def triples(t) -> set:
    return {tuple(int(v) for v in x) for x in np.asarray(t).reshape(-1, 3)}


def outside_window(diff, Ao, Bo, tau, na=None, nbn=None) -> list:
    """Triples of `diff` whose norm product is NOT within 1e-12 relative of T."""
    if not diff:
        return []
    na = Ao.leaf_norms() if na is None else na
    nbn = Bo.leaf_norms() if nbn is None else nbn
    thr = tau * Ao.norm() * Bo.norm()
    bad = []
    for (i, k, j) in diff:
        p = na[i, k] * nbn[k, j]
        if not (na[i, k] > 0 and nbn[k, j] > 0 and abs(p - thr) <= WINDOW * thr):
            bad.append((i, k, j))
    return bad


def flip_correct(oblocks: dict, Ao, Bo, only_gpu, only_oracle) -> dict:
    """The oracle's product with the flipped triples' contributions added / removed."""
    out = dict(oblocks)
    for sign, ts in ((1.0, only_gpu), (-1.0, only_oracle)):
        for (i, k, j) in ts:
            a, b = Ao.block(i, k), Bo.block(k, j)
            c = out.get((i, j))
            c = np.zeros_like(a) if c is None else c.copy()
            out[(i, j)] = c + sign * (a @ b)
    return out


def rel_union(gb: dict, ob: dict, keys=None) -> float:
    """||G - O||_F / ||O||_F over the union of stored blocks (or the given keys)."""
    keys = set(gb) | set(ob) if keys is None else keys
    num = den = 0.0
    for key in keys:
        g, o = gb.get(key), ob.get(key)
        if o is None:
            num += float(np.sum(g * g))
            continue
        den += float(np.sum(o * o))
        d = o if g is None else g - o
        num += float(np.sum(d * d))
    return math.sqrt(num) / (math.sqrt(den) if den > 0 else 1.0)
