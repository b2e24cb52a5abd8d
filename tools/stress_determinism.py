"""Determinism stress: fixed inputs (Y_4, Z_4), repeat Z (x) Y, the scaled and the plain NS step R times and
hash the outputs (every hash must occur R times).  python tools/stress_determinism.py R lib(0|1)"""
import collections, hashlib, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1508_05856_b200 as sp
import spamm_inputs as si
n, b = 4096, 64
R = int(sys.argv[1]); lib = bool(int(sys.argv[2]))
cfg = si.Config("t", "gauss", n, b, 1e-7, 30, sigma=0.8, shift=1e-3, seed=150805856, tau_min=1e-7)
payload = si.make_input(cfg)[1]
def h(ctx, M):
    bi, bj, blk = sp.spamm_export_blocks(ctx, M)
    o = np.lexsort((bj, bi))
    return hashlib.sha1(bi[o].tobytes() + bj[o].tobytes() + blk[o].tobytes()).hexdigest()[:10]
ctx = sp.spamm_ctx_create(0, library_stream=lib)
S = sp.spamm_build_tree_blocks(ctx, n, b, *payload)
Y = sp.spamm_ns_y0(ctx, S, 11.0); Z = sp.spamm_identity(ctx, n, b)
for k in range(4):
    Yn, Zn, t, st, ae = sp.spamm_ns_step_map(ctx, Y, Z, 1e-7, 1e-9, scaled=True)
    Y, Z = Yn, Zn
cnt = collections.defaultdict(collections.Counter)
for r in range(R):
    X = sp.spamm_multiply(ctx, Z, Y, 1e-7)
    cnt["X=ZY store"][h(ctx, X)] += 1
    X.free()
    Yn, Zn, t, st, ae, H = sp.spamm_ns_step_map(ctx, Y, Z, 1e-7, 1e-9, scaled=True, want_h=True)
    cnt["H scaled"][h(ctx, H)] += 1
    cnt["Y' scaled"][h(ctx, Yn)] += 1
    for m in (Yn, Zn, H): m.free()
    Yn, Zn, t, st, H = sp.spamm_ns_step(ctx, Y, Z, 1e-7, 1e-9, want_h=True)
    cnt["H plain"][h(ctx, H)] += 1
    for m in (Yn, Zn, H): m.free()
for k, v in cnt.items():
    print("lib" if lib else "torch", k, dict(v), flush=True)
