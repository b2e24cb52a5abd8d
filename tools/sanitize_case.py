"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck), SURVEY.md §4.5.

Exercises, on the library's own stream and cudaMallocAsync pool (no PyTorch caching
allocator, so memcheck sees every allocation's true bounds):
  * the leaf GEMM at b = 16, 32, 64 (k_leaf_gemm instances: store, NS-H, transposed-A);
  * the cull chain under programmatic dependent launch, both concurrent culls of an NS
    step (Y' on the context stream, Z' on the side stream);
  * the graph-replayed step (C1) and the host-driven step (C2), the scaled map, the
    single channel, the volume recorder and the asynchronous export.

  compute-sanitizer --tool memcheck python tools/sanitize_case.py [--quick]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1508_05856_b200 as sp  # noqa: E402
import spamm_inputs as si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    ctx = sp.spamm_ctx_create(0, library_stream=True)
    # C1 (b = 16): graph-replayed steps + the host-driven last step
    c1 = si.CONFIGS["C1"]
    S1 = sp.spamm_build_tree(ctx, si.kms(c1.n, c1.rho), c1.b)
    r = sp.spamm_ns_sqrt(ctx, S1, c1.tau, 8)
    print("C1 graph run t_last", r["t"][-1], flush=True)
    # C2 (b = 32): host-driven steps (volume sink disables the graph), concurrent culls
    c2 = si.CONFIGS["C2"]
    n2 = 1024 if a.quick else c2.n
    S2 = sp.spamm_build_tree(ctx, si.kms(n2, c2.rho), c2.b)
    sink = sp.VolumeSink(3 * 6, nbins=n2 // c2.b, ikj_cap=200000)
    sp.spamm_ctx_set_volume_sink(ctx, sink)
    r = sp.spamm_ns_sqrt(ctx, S2, c2.tau, 6)
    sp.spamm_ctx_set_volume_sink(ctx, None)
    print("C2 run t_last", r["t"][-1], "products", sink.nprod, flush=True)
    # scaled map and single channel on C1
    r = sp.spamm_ns_sqrt(ctx, S1, c1.tau, 6, scaled=True)
    r = sp.spamm_ns_sqrt_single(ctx, S1, c1.tau, 6)
    # b = 64 products: plain, transposed-left, and asynchronous export to host
    rng = np.random.default_rng(1)
    n = 512
    d = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :])
    A = sp.spamm_build_tree(ctx, np.exp(-0.02 * d) * rng.standard_normal((n, n)), 64)
    B = sp.spamm_build_tree(ctx, np.exp(-0.03 * d) * rng.standard_normal((n, n)), 64)
    C = sp.spamm_multiply(ctx, A, B, 1e-6)
    Ct = sp.spamm_multiply_t(ctx, A, B, 1e-6)
    out = (np.zeros(64, np.int32), np.zeros(64, np.int32), np.zeros((64, 64, 64)))
    k = sp.spamm_export_blocks_async(ctx, C, out)
    sp.spamm_copies_wait(ctx)
    print("b=64 products", C.nblocks, Ct.nblocks, "exported", k, flush=True)
    for m in (C, Ct, A, B, S1, S2):
        m.free()
    ctx.close()
    print("sanitize case done", flush=True)


if __name__ == "__main__":
    main()
