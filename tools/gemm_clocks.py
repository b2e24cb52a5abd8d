"""Where the leaf GEMM's consumer warps spend their cycles (diagnostic build with
-DSPAMM_GEMM_CLOCKS; built here if missing).  Runs k NS steps of a config, then one
more step with the counters reset, and prints per product role the share of the
consumer loop spent waiting for stages (full), for queue entries, and at segment
boundaries (the deposit in the epilogue warp's tile).

  python tools/gemm_clocks.py --config C5 -k 8
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1508_05856_b200 import _build  # noqa: E402

if "SPAMM_LIB" not in os.environ:
    os.environ["SPAMM_LIB"] = _build.build_clocks()

import torch  # noqa: E402

import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("-k", type=int, default=8)
a = ap.parse_args()
lib = sp.load()
fn = lib.spamm_debug_gemm_clocks
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()

cfg = si.CONFIGS[a.config]
tau, tau_s = cfg.tau, cfg.tau * cfg.tau_s_factor
kind, payload = si.make_input(cfg)
ctx = sp.spamm_ctx_create(0)
S = (sp.spamm_build_tree(ctx, torch.from_numpy(payload).cuda(), cfg.b) if kind == "dense" else
     sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *(torch.from_numpy(x).cuda() for x in payload)))
c = sp.spamm_power_scale(ctx, S, 100)
Y = sp.spamm_ns_y0(ctx, S, c, cfg.mu)
Z = sp.spamm_identity(ctx, cfg.n, cfg.b)
S.free()
for _ in range(a.k):
    Yn, Zn, _, _ = sp.spamm_ns_step(ctx, Y, Z, tau, tau_s)
    Y.free()
    Z.free()
    Y, Z = Yn, Zn
for name, (A, B) in (("Z*Y", (Z, Y)), ("Y*Z", (Y, Z)), ("Y*Y", (Y, Y))):
    fn(buf, 1)
    C, st = sp.spamm_multiply(ctx, A, B, tau, want_stats=True)
    torch.cuda.synchronize()
    fn(buf, 1)
    tot, full, q, bnd, nt, ns, cmap, cew = [float(x) for x in buf[:8]]
    print(f"{a.config} k={a.k} {name}: tasks {st['tasks']} segments {st['segments']} | per consumer warp-task "
          f"{tot / nt:.0f} clk: full-wait {full / tot:.2%} queue-wait {q / tot:.2%} boundary {bnd / tot:.2%} (map {cmap / tot:.2%}, tile wait {cew / tot:.2%}) "
          f"| tasks/seg {nt / max(ns, 1):.2f}", flush=True)
    C.free()
