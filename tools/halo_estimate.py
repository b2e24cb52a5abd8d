"""Multi-GPU cost model from one GPU: run the row-partitioned path with G in-process ranks
(threads, spamm_comm_local_group) and report, per product, each rank's leaf tasks and the
remote right-operand blocks its halo exchange fetched.  With the measured single-GPU GEMM
rate and an NVLink bandwidth this gives the per-rank compute / exchange balance that the
G-GPU run would see (the exchange is overlapped with the all-local segments)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1508_05856_b200 as sp  # noqa: E402
from paper_1508_05856_b200 import dist as D  # noqa: E402
import spamm_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--gpus", type=int, default=8)
ap.add_argument("--iters", type=int, default=16)
ap.add_argument("--gemm-tflops", type=float, default=33.0)
ap.add_argument("--nvlink-gbs", type=float, default=700.0)
a = ap.parse_args()
cfg = si.CONFIGS[a.config]
G, b = a.gpus, cfg.b
rs = D.equal_partition(cfg.n // b, G)


def fn(rank, comm):
    ctx = sp.spamm_ctx_create(0, library_stream=True)
    sp.spamm_ctx_set_comm(ctx, comm, rs)
    _, payload = si.make_input(cfg, rows=(rs[rank], rs[rank + 1]))
    S = sp.spamm_build_tree_blocks(ctx, cfg.n, b, *payload)
    r = sp.spamm_ns_sqrt(ctx, S, cfg.tau, a.iters, tau_s=cfg.tau * cfg.tau_s_factor, mu=cfg.mu,
                         t_stop=cfg.t_stop)
    out = np.array([[[p["tasks"], p["halo_blocks"], p["local_segments"], p["segments"]] for p in k]
                     for k in r["stats"]])
    for m in (S, r["Y"], r["Z"]):
        m.free()
    ctx.close()
    return out


res = np.stack(D.run_rank_threads(G, fn))          # [G, k, 3, 2]
tasks, halo = res[..., 0].astype(float), res[..., 1].astype(float)
loc_frac = res[..., 2].sum() / max(res[..., 3].sum(), 1)
flop_task, byte_blk = 2.0 * b ** 3, 8.0 * b * b
t_gemm = tasks * flop_task / (a.gemm_tflops * 1e12)       # per rank, per product
t_halo = halo * byte_blk / (a.nvlink_gbs * 1e9)
print(f"{a.config} G={G} equal split, {res.shape[1]} iterations; per-product maxima over ranks:")
for k in range(res.shape[1]):
    row = []
    for p, name in enumerate(("X=ZY", "Y'=YH", "Z'=HZ")):
        row.append(f"{name}: tasks {int(tasks[:, k, p].max()):7d} halo {halo[:, k, p].max() * byte_blk / 1e9:6.2f} GB "
                   f"gemm {1e3 * t_gemm[:, k, p].max():6.2f} ms xchg {1e3 * t_halo[:, k, p].max():6.2f} ms")
    print(f"k={k:2d} " + " | ".join(row))
tot_gemm = t_gemm.sum(axis=(1, 2)).max()
tot_serial = (t_gemm + t_halo).sum(axis=(1, 2)).max()
tot_overlap = np.maximum(t_gemm, t_halo).sum(axis=(1, 2)).max()
one = tasks.sum() * flop_task / (a.gemm_tflops * 1e12)
print(f"all-local segments (run while the halo is exchanged): {100 * loc_frac:.1f} % of all segments")
print(f"run GEMM time 1 GPU {one * 1e3:.1f} ms; G={G}: max-rank GEMM {tot_gemm * 1e3:.1f} ms, "
      f"+ exchange serial {tot_serial * 1e3:.1f} ms, overlapped {tot_overlap * 1e3:.1f} ms -> "
      f"efficiency {one / G / tot_serial:.2f} (serial) .. {one / G / tot_overlap:.2f} (perfect overlap)")
