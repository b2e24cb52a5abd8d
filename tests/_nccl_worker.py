"""torchrun worker of tests/test_gpu_nccl_multiprocess.py: one process per GPU, the
row-partitioned path over a real NCCL communicator.  Rank 0 also runs
the single-device reference and compares the gathered Y, Z and t_k bitwise."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402
from paper_1508_05856_b200 import dist as D  # noqa: E402


def digest(parts, t):
    rows = sorted((int(i), int(j), blk.tobytes()) for bi, bj, bl in parts for i, j, blk in zip(bi, bj, bl))
    h = hashlib.sha1(np.asarray(t).tobytes())
    for i, j, b in rows:
        h.update(np.int32([i, j]).tobytes() + b)
    return h.hexdigest()


def main():
    rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    cfg = si.Config("t", "gauss", 8192, 64, 1e-7, 30, sigma=0.8, shift=1e-3, seed=150805856, tau_min=1e-7)
    payload = si.make_input(cfg)[1]
    iters = 12
    comm = D.init_nccl_comm(local)
    ctx = sp.spamm_ctx_create(local)
    sp.spamm_ctx_set_comm(ctx, comm)
    S = sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *(torch.from_numpy(x).to(dev) for x in payload))
    r = sp.spamm_ns_sqrt(ctx, S, cfg.tau, iters, tau_s=1e-9)
    mine = [sp.spamm_export_blocks(ctx, r[k]) for k in ("Y", "Z")]
    halo = [p["halo_blocks"] for k in r["stats"] for p in k]
    allY = D.gather_to_rank0(mine[0])
    allZ = D.gather_to_rank0(mine[1])
    halos = D.gather_to_rank0(int(sum(halo)))
    t = r["t"].copy()
    if rank == 0:
        c1 = sp.spamm_ctx_create(local)
        S1 = sp.spamm_build_tree_blocks(c1, cfg.n, cfg.b, *(torch.from_numpy(x).to(dev) for x in payload))
        r1 = sp.spamm_ns_sqrt(c1, S1, cfg.tau, iters, tau_s=1e-9)
        ok = (digest(allY, t) == digest([sp.spamm_export_blocks(c1, r1["Y"])], r1["t"]) and
              digest(allZ, t) == digest([sp.spamm_export_blocks(c1, r1["Z"])], r1["t"]))
        print(f"NCCL world {ws}: bitwise equal to G=1: {ok}; halo blocks per rank {halos}", flush=True)
        if not ok:
            sys.exit(1)
    ctx.close()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
