"""Load balance of row partitions for the multi-GPU path: per-row leaf task counts of the
three products at NS iteration k (one GPU), and the max/mean per-rank load for the equal
split and for the split balanced on s (x)_tau s (what bench.py --partition balanced uses)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1508_05856_b200 as sp  # noqa: E402
from paper_1508_05856_b200 import dist as D  # noqa: E402
import spamm_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--ks", default="0,4,8,12,15")
a = ap.parse_args()
cfg = si.CONFIGS[a.config]
tau, tau_s = cfg.tau, cfg.tau * cfg.tau_s_factor
_, payload = si.make_input(cfg)
ctx = sp.spamm_ctx_create(0)
S = sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *(torch.from_numpy(x).cuda() for x in payload))
proxy = sp.spamm_row_task_counts(ctx, S, S, tau)
c = sp.spamm_power_scale(ctx, S, 100)
Y, Z = sp.spamm_ns_y0(ctx, S, c, cfg.mu), sp.spamm_identity(ctx, cfg.n, cfg.b)
ks = [int(x) for x in a.ks.split(",")]
for k in range(max(ks) + 1):
    Yn, Zn, t, st, H = sp.spamm_ns_step(ctx, Y, Z, tau, tau_s, want_h=True)
    if k in ks:
        rows = sp.spamm_row_task_counts(ctx, Z, Y, tau) + sp.spamm_row_task_counts(ctx, Y, H, tau_s) + \
            sp.spamm_row_task_counts(ctx, H, Z, tau)
        for G in (2, 4, 8):
            eq, bal = D.equal_partition(len(rows), G), D.balanced_partition(proxy, G)
            le, lb = D.partition_loads(rows, eq), D.partition_loads(rows, bal)
            print(f"k={k:2d} G={G}: max/mean equal {max(le) / np.mean(le):.3f}  balanced(s*s) {max(lb) / np.mean(lb):.3f}"
                  f"  ideal(this k) {max(D.partition_loads(rows, D.balanced_partition(rows, G))) / np.mean(le):.3f}",
                  flush=True)
    H.free()
    Y.free()
    Z.free()
    Y, Z = Yn, Zn
