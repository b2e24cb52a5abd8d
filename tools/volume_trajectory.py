"""Per-product ijk volume trajectory of a dual NS run.

The paper's locality / lensing evidence is per iteration and per product: the
volumes of the x_k and y_k products at several k (Figs. Lensing1-3) and
"locality increases compressively towards convergence".  This runs
spamm_ns_sqrt on the GPU with the library's per-product volume recorder
(spamm_ctx_set_volume_sink) and prints, for every k and product (X = Z(x)Y,
Y' = Y(x)H, Z' = H(x)Z): the task count |S| (the volume) and the
distribution of the diagonal-plane distance d = max(|i-j|, |i-k|, |j-k|):
its quantiles and the share of the volume within d <= 1, 2, 4.

  python tools/volume_trajectory.py --config C2 [--iters 30] [--tau-s 1e-10]
                                    [--vtk DIR --vtk-k 0,5,17]

--vtk writes the chosen steps' ijk volumes as legacy-VTK point clouds (one vertex
per surviving leaf triple, scalar d), the "sparse VTK output for visualization of
the ijk product volumes" of P:418-419.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402

PRODUCTS = ("X", "Y'", "Z'")


def quantile_of_hist(h, q):
    c = np.cumsum(h)
    return int(np.searchsorted(c, q * c[-1])) if c[-1] else 0


def write_vtk(path, ikj, title):
    d = np.max(np.abs(np.stack([ikj[:, 0] - ikj[:, 2], ikj[:, 0] - ikj[:, 1], ikj[:, 2] - ikj[:, 1]])), axis=0)
    n = len(ikj)
    with open(path, "w") as f:
        f.write(f"# vtk DataFile Version 3.0\n{title}\nASCII\nDATASET POLYDATA\nPOINTS {n} int\n")
        np.savetxt(f, ikj[:, [0, 1, 2]], fmt="%d")
        f.write(f"VERTICES {n} {2 * n}\n")
        np.savetxt(f, np.stack([np.ones(n, dtype=np.int64), np.arange(n)], axis=1), fmt="%d")
        f.write(f"POINT_DATA {n}\nSCALARS d int 1\nLOOKUP_TABLE default\n")
        np.savetxt(f, d, fmt="%d")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--tau", type=float, default=None)
    ap.add_argument("--tau-s", type=float, default=None)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--json", default=None, help="write the table as JSON here")
    ap.add_argument("--vtk", default=None, help="directory for VTK point clouds")
    ap.add_argument("--vtk-k", default="0,5,17")
    a = ap.parse_args()
    cfg = si.CONFIGS[a.config]
    tau = a.tau if a.tau is not None else cfg.tau
    tau_s = a.tau_s if a.tau_s is not None else tau * cfg.tau_s_factor
    iters = a.iters or cfg.iters
    kind, payload = si.make_input(cfg)
    ctx = sp.spamm_ctx_create(0)
    if kind == "dense":
        S = sp.spamm_build_tree(ctx, torch.from_numpy(payload).cuda(), cfg.b)
    else:
        S = sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *(torch.from_numpy(x).cuda() for x in payload))
    nb = cfg.n // cfg.b
    vtk_k = {int(x) for x in a.vtk_k.split(",")} if a.vtk else set()
    # pass 1: counts and histograms for every product; pass 2 (only with --vtk): triples
    sink = sp.VolumeSink(3 * iters, nbins=nb)
    sp.spamm_ctx_set_volume_sink(ctx, sink)
    r = sp.spamm_ns_sqrt(ctx, S, tau, iters, tau_s=tau_s, mu=cfg.mu, t_stop=cfg.t_stop)
    sp.spamm_ctx_set_volume_sink(ctx, None)
    rows = []
    print(f"{a.config} n={cfg.n} b={cfg.b} tau={tau} tau_s={tau_s} iters run={r['iters']}")
    print(f"{'k':>3} {'prod':>4} {'tasks':>10} {'d50':>5} {'d90':>5} {'d99':>5} {'<=1':>7} {'<=2':>7} {'<=4':>7}")
    for p in range(sink.nprod):
        k, q = divmod(p, 3)
        h = sink.hist[p]
        tot = max(int(h.sum()), 1)
        row = dict(k=k, product=PRODUCTS[q], tasks=int(sink.ntasks[p]), t=float(r["t"][k]),
                   d50=quantile_of_hist(h, 0.5), d90=quantile_of_hist(h, 0.9), d99=quantile_of_hist(h, 0.99),
                   le1=float(h[:2].sum() / tot), le2=float(h[:3].sum() / tot), le4=float(h[:5].sum() / tot))
        rows.append(row)
        print(f"{k:3d} {row['product']:>4} {row['tasks']:10d} {row['d50']:5d} {row['d90']:5d} {row['d99']:5d} "
              f"{row['le1']:7.3f} {row['le2']:7.3f} {row['le4']:7.3f}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(dict(config=a.config, n=cfg.n, b=cfg.b, tau=tau, tau_s=tau_s, iters=int(r["iters"]),
                           rows=rows), f, indent=1)
    if vtk_k:
        os.makedirs(a.vtk, exist_ok=True)
        need = int(sum(sink.ntasks[3 * k + q] for k in vtk_k if 3 * k + 2 < sink.nprod for q in range(3)))
        total = int(sink.ntasks.sum())
        full = sp.VolumeSink(3 * iters, ikj_cap=total)
        sp.spamm_ctx_set_volume_sink(ctx, full)
        sp.spamm_ns_sqrt(ctx, S, tau, iters, tau_s=tau_s, mu=cfg.mu, t_stop=cfg.t_stop)
        sp.spamm_ctx_set_volume_sink(ctx, None)
        assert full.complete() and np.array_equal(full.ntasks, sink.ntasks)
        for k in sorted(vtk_k):
            for q in range(3):
                p = 3 * k + q
                if p < full.nprod:
                    fn = os.path.join(a.vtk, f"{a.config}_k{k:02d}_{'XYZ'[q]}.vtk")
                    write_vtk(fn, full.tasks(p), f"{a.config} k={k} {PRODUCTS[q]} ijk volume")
        print(f"wrote VTK volumes for k in {sorted(vtk_k)} ({need} triples) to {a.vtk}")


if __name__ == "__main__":
    main()
