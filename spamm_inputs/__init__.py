"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module holds NO arithmetic of the SpAMM method (no norms of the method's
quadtree, no culling, no products, no Newton-Schulz). It only produces the
input matrices that stand in for the paper's data (§4.3 "Data",
P:451-466), as the BASELINE.json configs define them:

* KMS Toeplitz matrices  s_ij = rho^|i-j|             (BJ:7, BJ:8)
* 3-D Gaussian-overlap matrices on Hilbert-ordered points (BJ:9-11),
  s_ij = exp(-|r_i - r_j|^2 / (2 sigma^2)) + shift * delta_ij,
  generated block-sparse with the lossless drop rule of DESIGN.md §3.

Both `oracle/` and `paper_1508_05856_b200/` consume the bits produced here;
neither side recomputes an input.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "kms",
    "splitmix64",
    "uniform_points",
    "hilbert_keys",
    "hilbert_order",
    "gaussian_blocks",
    "gaussian_dense",
    "blocks_to_dense",
    "Config",
    "CONFIGS",
    "make_input",
]

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def kms(n: int, rho: float) -> np.ndarray:
    """Kac-Murdock-Szegő matrix s_ij = rho^|i-j| (BJ:7-8), dense fp64 row-major."""
    idx = np.arange(n)
    d = np.abs(idx[:, None] - idx[None, :]).astype(np.float64)
    return np.ascontiguousarray(np.power(np.float64(rho), d))


def splitmix64(seed: int, count: int) -> np.ndarray:
    """The splitmix64 stream: x_i = mix(seed + (i+1)*gamma), i = 0..count-1 (uint64)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_points(n: int, seed: int, box: float) -> np.ndarray:
    """n points i.i.d. uniform in [0, box)^3: point i uses draws 3i, 3i+1, 3i+2,
    u = (x >> 11) * 2^-53 (SURVEY §8(d) recipe)."""
    x = splitmix64(seed, 3 * n)
    u = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (u * box).reshape(n, 3)


def _axes_to_transpose(X: np.ndarray, bits: int) -> np.ndarray:
    """Skilling's 'AxestoTranspose' (AIP Conf. Proc. 707, 2004) vectorised over
    rows of X (shape [npts, ndim], non-negative ints < 2^bits)."""
    X = X.astype(np.uint64).copy()
    ndim = X.shape[1]
    M = np.uint64(1 << (bits - 1))
    # inverse undo
    Q = M
    while Q > 1:
        P = Q - np.uint64(1)
        for i in range(ndim):
            hit = (X[:, i] & Q) != 0
            # if bit set: invert low bits of X[0]
            X[hit, 0] ^= P
            # else: exchange low bits of X[0] and X[i]
            nh = ~hit
            t = (X[nh, 0] ^ X[nh, i]) & P
            X[nh, 0] ^= t
            X[nh, i] ^= t
        Q >>= np.uint64(1)
    # Gray encode
    for i in range(1, ndim):
        X[:, i] ^= X[:, i - 1]
    t = np.zeros(X.shape[0], dtype=np.uint64)
    Q = M
    while Q > 1:
        hit = (X[:, ndim - 1] & Q) != 0
        t[hit] ^= Q - np.uint64(1)
        Q >>= np.uint64(1)
    for i in range(ndim):
        X[:, i] ^= t
    return X


def hilbert_keys(cells: np.ndarray, bits: int) -> np.ndarray:
    """Hilbert index of integer cells [npts, ndim] with `bits` bits per axis
    (transpose form interleaved most-significant bit first, axis 0 first)."""
    T = _axes_to_transpose(np.asarray(cells), bits)
    ndim = T.shape[1]
    key = np.zeros(T.shape[0], dtype=np.uint64)
    for b in range(bits - 1, -1, -1):
        for i in range(ndim):
            key = (key << np.uint64(1)) | ((T[:, i] >> np.uint64(b)) & np.uint64(1))
    return key


def hilbert_order(points: np.ndarray, box: float, bits: int = 16) -> np.ndarray:
    """Permutation sorting points along the Hilbert curve: 16-bit-per-axis
    quantisation of r/box, stable tie-break by generation index (reading L18)."""
    q = np.floor(points / box * (1 << bits)).astype(np.int64)
    q = np.clip(q, 0, (1 << bits) - 1)
    keys = hilbert_keys(q, bits)
    return np.argsort(keys, kind="stable")


def _block_bboxes(pts: np.ndarray, b: int):
    nb = pts.shape[0] // b
    p = pts.reshape(nb, b, 3)
    return p.min(axis=1), p.max(axis=1)


def gaussian_blocks(points: np.ndarray, b: int, sigma: float, shift: float,
                    delta: float, rows=None):
    """Block-sparse Gaussian overlap s_IJ (b x b blocks) for Hilbert-ordered points.

    Candidate block pair (I,J) is skipped when b*exp(-dmin^2/(2 sigma^2)) < delta
    (dmin: distance between the blocks' point bounding boxes, an upper bound on
    every |s_ij| of the block, so ||s_IJ||_F <= b*max|s_ij| < delta), otherwise it
    is computed and kept iff ||s_IJ||_F >= delta.  Returns (bi, bj, blocks) with
    blocks [nblk, b, b] fp64, ordered by (bi, bj).  rows = (r0, r1) generates only
    block rows r0 <= I < r1 (a rank's shard of the row partition; the blocks are
    bitwise those of the full generation)."""
    n = points.shape[0]
    assert n % b == 0
    nb = n // b
    lo, hi = _block_bboxes(points, b)
    inv2s2 = 1.0 / (2.0 * sigma * sigma)
    out_i, out_j, out_b = [], [], []
    P = points.reshape(nb, b, 3)
    r0, r1 = (0, nb) if rows is None else rows
    for I in range(r0, r1):
        gap = np.maximum(0.0, np.maximum(lo[I][None, :] - hi, lo - hi[I][None, :]))
        dmin2 = np.sum(gap * gap, axis=1)
        cand = np.nonzero(b * np.exp(-dmin2 * inv2s2) >= delta)[0]
        if cand.size == 0:
            continue
        ri = P[I]                                   # [b,3]
        rj = P[cand]                                # [c,b,3]
        d = ri[None, :, None, :] - rj[:, None, :, :]  # [c,b,b,3]
        d2 = np.sum(d * d, axis=-1)
        blk = np.exp(-d2 * inv2s2)
        diag = np.nonzero(cand == I)[0]
        if diag.size:
            blk[diag[0]] += shift * np.eye(b)
        fro = np.sqrt(np.sum(blk * blk, axis=(1, 2)))
        keep = fro >= delta
        if np.any(keep):
            out_i.append(np.full(int(keep.sum()), I, dtype=np.int32))
            out_j.append(cand[keep].astype(np.int32))
            out_b.append(blk[keep])
    if not out_i:
        return np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, b, b))
    bi = np.concatenate(out_i)
    bj = np.concatenate(out_j)
    blocks = np.ascontiguousarray(np.concatenate(out_b, axis=0))
    return bi, bj, blocks


def gaussian_dense(points: np.ndarray, sigma: float, shift: float) -> np.ndarray:
    """Dense Gaussian overlap (small n only)."""
    d = points[:, None, :] - points[None, :, :]
    s = np.exp(-np.sum(d * d, axis=-1) / (2.0 * sigma * sigma))
    s += shift * np.eye(points.shape[0])
    return s


def blocks_to_dense(n: int, b: int, bi, bj, blocks) -> np.ndarray:
    s = np.zeros((n, n))
    for I, J, blk in zip(bi, bj, blocks):
        s[I * b:(I + 1) * b, J * b:(J + 1) * b] = blk
    return s


@dataclass(frozen=True)
class Config:
    name: str
    kind: str            # "kms" | "gauss"
    n: int
    b: int
    tau: float
    iters: int
    rho: float = 0.0
    sigma: float = 0.0
    shift: float = 0.0
    mu: float = 0.0
    seed: int = 0
    tau_min: float = 0.0  # smallest tau the input must serve (drop rule)
    # run options (readings L9, L15): tau_s = tau_s_factor * tau; t_stop > 0
    # ends the run at convergence (|t_k| <= t_stop) instead of after `iters`
    tau_s_factor: float = 1.0
    t_stop: float = 0.0


# BASELINE.json configs[0..4] (BJ:7-11); C4's tau sweep is {1e-4,1e-6,1e-8}.
CONFIGS = {
    "C1": Config("C1", "kms", 256, 16, 1e-6, 25, rho=0.5),
    "C2": Config("C2", "kms", 4096, 32, 1e-8, 30, rho=0.9),
    "C3": Config("C3", "gauss", 16384, 64, 1e-7, 30, sigma=0.8, shift=1e-3,
                 seed=150805856, tau_min=1e-7),
    # C4 / C5: with tau_s = tau the plain dual iteration diverges (C4 tau = 1e-6 at
    # k = 14, C5 at k = 10; profiles/r01_diag), so these use the paper's default
    # sensitive threshold tau_s = .01 tau and stop at convergence.
    "C4": Config("C4", "gauss", 32768, 64, 1e-6, 40, sigma=1.2, shift=0.0,
                 mu=1e-2, seed=150805857, tau_min=1e-8, tau_s_factor=0.01, t_stop=1e-5),
    "C5": Config("C5", "gauss", 131072, 64, 1e-7, 30, sigma=0.8, shift=1e-3,
                 seed=150805858, tau_min=1e-7, tau_s_factor=0.01, t_stop=1e-5),
}


def make_input(cfg: Config, n: int | None = None, rows=None):
    """Return ("dense", s) for KMS configs or ("blocks", (bi, bj, blocks)) for the
    Gaussian configs.  `n` overrides the dimension (scaled-down parity cases);
    the box keeps unit density, L = n^(1/3).  `rows` = (r0, r1) restricts the
    Gaussian block list to block rows [r0, r1) (KMS inputs are returned whole)."""
    n = cfg.n if n is None else n
    if cfg.kind == "kms":
        return "dense", kms(n, cfg.rho)
    box = n ** (1.0 / 3.0)
    pts = uniform_points(n, cfg.seed, box)
    pts = np.ascontiguousarray(pts[hilbert_order(pts, box)])
    delta = 1e-2 * cfg.tau_min * math.sqrt(n)
    return "blocks", gaussian_blocks(pts, cfg.b, cfg.sigma, cfg.shift, delta, rows)
