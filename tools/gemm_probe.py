"""A/B timing of single SpAMM products on realistic iterates: runs k dual NS steps of a config,
then times spamm_multiply(Z, Y) (the X product's task set, plain store epilogue) and
spamm_multiply(Y, Z) with CUDA events (cull + GEMM), best of --reps.
SPAMM_LIB=<path> selects an experimental build of the library."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("-k", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dense", type=int, default=0, help="instead: dense random n x n (b = 64), tau = 0")
a = ap.parse_args()


def timed(ctx, A, B, tau, reps):
    best, st = 1e30, None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream) if ctx.stream is not None else e0.record()
        C, st = sp.spamm_multiply(ctx, A, B, tau, want_stats=True)
        e1.record(ctx.stream) if ctx.stream is not None else e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
        C.free()
    return best, st


if a.dense:
    ctx = sp.spamm_ctx_create(0)
    g = torch.Generator().manual_seed(1)
    M = sp.spamm_build_tree(ctx, torch.randn(a.dense, a.dense, generator=g, dtype=torch.float64).cuda(), 64)
    for _ in range(2):
        best, st = timed(ctx, M, M, 0.0, a.reps)
        print(f"dense n={a.dense}: tasks {st['tasks']} segments {st['segments']} "
              f"({st['tasks'] / max(st['segments'], 1):.1f} per segment) {best:.3f} ms "
              f"{st['flops'] / best / 1e9:.2f} TFLOP/s", flush=True)
    sys.exit(0)
cfg = si.CONFIGS[a.config]
tau, tau_s = cfg.tau, cfg.tau * cfg.tau_s_factor
kind, payload = si.make_input(cfg)
ctx = sp.spamm_ctx_create(0)
if kind == "dense":
    S = sp.spamm_build_tree(ctx, torch.from_numpy(payload).cuda(), cfg.b)
else:
    S = sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *(torch.from_numpy(x).cuda() for x in payload))
c = sp.spamm_power_scale(ctx, S, 100)
Y = sp.spamm_ns_y0(ctx, S, c, cfg.mu)
Z = sp.spamm_identity(ctx, cfg.n, cfg.b)
S.free()
for _ in range(a.k):
    Yn, Zn, _, _ = sp.spamm_ns_step(ctx, Y, Z, tau, tau_s)
    Y.free()
    Z.free()
    Y, Z = Yn, Zn
for name, (A, B) in (("Z*Y", (Z, Y)), ("Y*Z", (Y, Z))):
    best, st = timed(ctx, A, B, tau, a.reps)
    print(f"{a.config} k={a.k} {name}: tasks {st['tasks']} segments {st['segments']} "
          f"({st['tasks'] / max(st['segments'], 1):.2f} per segment) {best:.3f} ms "
          f"{st['flops'] / best / 1e9:.2f} TFLOP/s", flush=True)
# one whole NS step (X with the fused H epilogue, Y', Z'): GEMM time per product from the
# library's phase events, best of --reps
best = None
for _ in range(a.reps):
    sp.spamm_profile_enable(ctx, True)
    Yn, Zn, t, st = sp.spamm_ns_step(ctx, Y, Z, tau, tau_s)
    torch.cuda.synchronize()
    prof = sp.spamm_profile_read(ctx)
    sp.spamm_profile_enable(ctx, False)
    Yn.free()
    Zn.free()
    if best is None or prof["gemm_ms"] < best[0]["gemm_ms"]:
        best = (prof, st)
prof, st = best
fl = sum(p["flops"] for p in st)
print(f"{a.config} k={a.k} NS step: tasks {[p['tasks'] for p in st]} GEMM {prof['gemm_ms']:.3f} ms "
      f"({prof['gemm_count']} launches) {fl / prof['gemm_ms'] / 1e9:.2f} TFLOP/s", flush=True)
