"""Per-iteration trace of the dual NS run on the GPU: t_k, ||Y||_F, ||Z||_F and the
three task counts per k (diagnostics for divergence at large n / loose tau).

  python tools/diag_ns.py --config C5 [--tau 1e-7] [--iters 30] [--n 32768]
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--tau", type=float, default=None)
    ap.add_argument("--tau-s", type=float, default=None)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    cfg = si.CONFIGS[a.config]
    tau = a.tau if a.tau is not None else cfg.tau
    iters = a.iters or cfg.iters
    kind, payload = si.make_input(cfg, a.n)
    n = a.n or cfg.n
    ctx = sp.spamm_ctx_create(0)
    if kind == "dense":
        S = sp.spamm_build_tree(ctx, torch.from_numpy(payload).cuda(), cfg.b)
    else:
        S = sp.spamm_build_tree_blocks(ctx, n, cfg.b, *(torch.from_numpy(x).cuda() for x in payload))
    c = sp.spamm_power_scale(ctx, S, 100)
    print(f"{a.config} n={n} b={cfg.b} tau={tau} mu={cfg.mu} blocks(s)={S.nblocks} "
          f"||s||_F={sp.spamm_norm(ctx, S):.6e} c={c:.9e} T/(|Y||H|)~tau*n={tau * n:.3e}", flush=True)
    Y = sp.spamm_ns_y0(ctx, S, c, cfg.mu)
    Z = sp.spamm_identity(ctx, n, cfg.b)
    for k in range(iters):
        try:
            Yn, Zn, t, st = sp.spamm_ns_step(ctx, Y, Z, tau, a.tau_s)
        except sp.SpammError as e:
            print(f"k={k}: {e}", flush=True)
            break
        print(f"k={k:2d} t={t:+.6e} |Y|={sp.spamm_norm(ctx, Yn):.6e} |Z|={sp.spamm_norm(ctx, Zn):.6e} "
              f"tasks={[s['tasks'] for s in st]} blocks Y={Yn.nblocks} Z={Zn.nblocks}", flush=True)
        if not math.isfinite(t):
            break
        Y.free()
        Z.free()
        Y, Z = Yn, Zn


if __name__ == "__main__":
    main()
