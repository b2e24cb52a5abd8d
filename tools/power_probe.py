"""Time spamm_power_scale (K = 100) on a config's s: `python tools/power_probe.py C2`."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1508_05856_b200 as sp
import spamm_inputs as si

c = si.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
kind, p = si.make_input(c)
ctx = sp.spamm_ctx_create(0)
S = (sp.spamm_build_tree_blocks(ctx, c.n, c.b, *(torch.from_numpy(x).cuda() for x in p))
     if kind == "blocks" else sp.spamm_build_tree(ctx, torch.from_numpy(p).cuda(), c.b))
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cval = sp.spamm_power_scale(ctx, S, 100)
    torch.cuda.synchronize()
    print(f"{sys.argv[1:]} power_scale {1e3 * (time.perf_counter() - t0):.3f} ms c={cval!r}")
