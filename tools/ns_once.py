"""One full spamm_ns_sqrt run of a config (after one warm-up run that captures the graphs):
`python tools/ns_once.py C2` — for ncu launch lists of the small configs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402

cfg = si.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
kind, p = si.make_input(cfg)
ctx = sp.spamm_ctx_create(0)
S = (sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *(torch.from_numpy(x).cuda() for x in p))
     if kind == "blocks" else sp.spamm_build_tree(ctx, torch.from_numpy(p).cuda(), cfg.b))
for rep in range(2):
    r = sp.spamm_ns_sqrt(ctx, S, cfg.tau, cfg.iters, tau_s=cfg.tau * cfg.tau_s_factor, mu=cfg.mu)
    torch.cuda.synchronize()
    print(f"{cfg.name} run {rep}: t_last {r['t'][-1]:.3e}")
    r["Y"].free()
    r["Z"].free()
