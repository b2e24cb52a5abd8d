"""Time spamm_power_scale (K = 100) on the C1 / C2 inputs with CUDA events, best of 5
(A/B of SPAMM_POWER_FUSED in separate processes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402

ctx = sp.spamm_ctx_create(0)
for name in ("C1", "C2"):
    c = si.CONFIGS[name]
    S = sp.spamm_build_tree(ctx, si.kms(c.n, c.rho), c.b)
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        val = sp.spamm_power_scale(ctx, S, 100)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name} fused={os.environ.get('SPAMM_POWER_FUSED', '1')} power_scale(K=100) {best:.3f} ms c={val!r}",
          flush=True)
