import sys, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_1508_05856_b200 as sp, spamm_inputs as si
lib = int(sys.argv[1])
cfg = si.CONFIGS['C5']; n, b = cfg.n, cfg.b
_, (bi, bj, blocks) = si.make_input(cfg)
ctx = sp.spamm_ctx_create(0, library_stream=bool(lib))
dev = torch.device('cuda:0')
S = sp.spamm_build_tree_blocks(ctx, n, b, *(torch.from_numpy(x).to(dev) for x in (bi, bj, blocks)))
c = sp.spamm_power_scale(ctx, S, 100)
Y = sp.spamm_ns_y0(ctx, S, c, cfg.mu); Z = sp.spamm_identity(ctx, n, b)
S.free()
print('c', c, 'Y blocks', Y.nblocks, flush=True)
for k in range(2):
    Yn, Zn, t, st = sp.spamm_ns_step(ctx, Y, Z, cfg.tau, cfg.tau * cfg.tau_s_factor)
    print(k, t, [s['tasks'] for s in st], flush=True)
    Y, Z = Yn, Zn
