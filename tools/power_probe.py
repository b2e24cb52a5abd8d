"""Time spamm_power_scale (K SpMV + normalisations) on a config's s, CUDA events.
SPAMM_SPMV_SYM=0/1/2 selects the full / symmetric SpMV (read once per process)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("-K", type=int, default=100)
a = ap.parse_args()
cfg = si.CONFIGS[a.config]
kind, payload = si.make_input(cfg)
ctx = sp.spamm_ctx_create(0)
if kind == "dense":
    S = sp.spamm_build_tree(ctx, torch.from_numpy(payload).cuda(), cfg.b)
else:
    S = sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *(torch.from_numpy(x).cuda() for x in payload))
c0 = sp.spamm_power_scale(ctx, S, a.K)
ts = []
for _ in range(a.reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = sp.spamm_power_scale(ctx, S, a.K)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    assert c == c0
print(f"{a.config} sym={os.environ.get('SPAMM_SPMV_SYM', '1')} c={c0!r} power_scale K={a.K}: "
      f"{min(ts):.3f} ms (per SpMV+norm {min(ts) / (a.K + 1) * 1e3:.1f} us)")
