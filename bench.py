#!/usr/bin/env python
"""bench.py — SpAMM dual Newton-Schulz on B200 (arXiv 1508.05856 hot path).

One "step" = one full pass of the hot path over the
synthetic input: quadtree build of s from its block list, power-iteration
scale, Y0 = s/c, Z0 = I, `iters` dual NS iterations (3 SpAMM products each:
cull + FP64 DMMA leaf GEMM + fused epilogues + norm pyramids) and the unscale.

metric (BASELINE.json): culled-leaf FP64 TFLOP/s = sum over products of
|S| * 2 b^3 / time (only surviving leaf tasks count), plus seconds per NS
iteration.  `value` is timed with CUDA events on the library stream with the
inputs already resident in HBM; `e2e` repeats the step through the C ABI with
pinned HOST input buffers (H2D inside the timed region) and reads Y and Z back
to the host every step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import spamm_inputs as si  # noqa: E402

METRIC = "SpAMM culled-leaf FP64 TFLOP/s and seconds per Newton-Schulz step, 1/2/4/8 GPU"
UNIT = "TFLOP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    # C5 is the configuration BASELINE.json partitions across 1/2/4/8 GPUs (BJ:11) and
    # it fits one B200; C3 (BJ:9) is the other throughput config (--config C3)
    ap.add_argument("--config", default="C5", choices=sorted(si.CONFIGS))
    ap.add_argument("--tau", type=float, default=None, help="override tau (C4 sweep)")
    ap.add_argument("--iters", type=int, default=None, help="override NS iterations")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--map", default="plain", choices=["plain", "scaled"],
                    help="NS map: plain 1/2(3I-X) (north_star) or the paper's scaled/stabilised h_alpha")
    ap.add_argument("--channel", default="dual", choices=["dual", "single"],
                    help="dual (north_star, P:383-389) or single-channel (P:398-402) iteration")
    ap.add_argument("--tau-s-factor", type=float, default=None, help="override tau_s / tau")
    ap.add_argument("--t-stop", type=float, default=None, help="override the convergence exit |t_k| <= t_stop")
    ap.add_argument("--allocator", default="torch", choices=["torch", "cuda"],
                    help="device memory: PyTorch's caching allocator (callbacks) or cudaMallocAsync")
    ap.add_argument("--partition", default="equal", choices=["equal", "balanced"],
                    help="row partition for --gpus > 1 (balanced: on s (x) s per-row task counts)")
    ap.add_argument("--dist-world1", action="store_true",
                    help="run the row-partitioned NCCL path even at world size 1 (path check)")
    ap.add_argument("--ref-iters", type=int, default=1,
                    help="NS iterations of one oracle sample step (reference arm / cpu_baseline)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((num(r[3]) or 0) for r in rows)}


# --------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_name(cfg, tau, iters):
    if cfg.kind == "kms":
        return (f"{cfg.name}: KMS s_ij={cfg.rho}^|i-j|, N={cfg.n}, leaf {cfg.b}, tau={tau:g}, "
                f"{iters} dual NS iterations")
    return (f"{cfg.name}: 3-D Gaussian overlap, N={cfg.n} Hilbert-ordered unit-density points, "
            f"sigma={cfg.sigma}, shift={cfg.shift:g}, mu={cfg.mu:g}, leaf {cfg.b}, tau={tau:g}, "
            f"{iters} dual NS iterations")


def cpu_model():
    """lscpu model name / sockets / cores of this host (SURVEY.md §8(d) oracle timing)."""
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            info[k.strip()] = v.strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"model": info.get("Model name"), "sockets": info.get("Socket(s)"),
            "cores_per_socket": info.get("Core(s) per socket"), "threads": os.cpu_count()}


def oracle_sample(cfg, payload, tau, iters, scale, tau_s=None):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload:
    build + Y0 (given scale) + `iters` NS iterations, each NS iteration timed on its
    own.  Returns (seconds, flops, threads, per_k_seconds, build_seconds)."""
    import oracle as O
    t0 = time.perf_counter()
    if cfg.kind == "kms":
        So = O.OMat.from_dense(payload, cfg.b)
    else:
        So = O.OMat.from_blocks(cfg.n, cfg.b, *payload)
    Y, Z = O.ns_y0(So, scale, cfg.mu), O.OMat.identity(cfg.n, cfg.b)
    del So
    t1 = time.perf_counter()
    flops, per_k = 0.0, []
    for _ in range(iters):
        tk = time.perf_counter()
        Y, Z, _, _, counts = O.ns_step(Y, Z, tau, tau_s, allow_nonfinite=True)
        per_k.append(time.perf_counter() - tk)
        flops += float(counts.sum()) * 2.0 * cfg.b ** 3
    dt = time.perf_counter() - t0
    return dt, flops, O.num_threads(), per_k, t1 - t0


def run_config(args, cfg, ws, in_bytes):
    """The `config` object of the JSON line, identical for both arms at the same flags and N."""
    tau = args.tau if args.tau is not None else cfg.tau
    iters = args.iters if args.iters is not None else cfg.iters
    tau_s = tau * (args.tau_s_factor if args.tau_s_factor is not None else cfg.tau_s_factor)
    t_stop = args.t_stop if args.t_stop is not None else cfg.t_stop
    dist_path = ws > 1 or args.dist_world1
    return {
        "workload": workload_name(cfg, tau, iters), "n": cfg.n, "leaf": cfg.b, "tau": tau,
        "tau_s": tau_s, "iters": iters, "t_stop": t_stop, "map": args.map, "channel": args.channel,
        "parallelism": (f"row-partitioned over {ws} GPUs ({args.partition} split), NCCL halo "
                        "exchange + norm all-gather") if dist_path else "single",
        "l2": (f"inputs larger than L2 (s ~ {in_bytes / 1e6:.0f} MB of blocks, iterates > 126 MB)"
               if in_bytes > 126e6 else
               f"s ~ {in_bytes / 1e6:.1f} MB fits in L2, no flush between steps (latency-bound parity "
               "config, not the bench workload)"),
    }


def payload_bytes(kind, payload):
    return payload.nbytes if kind == "dense" else sum(x.nbytes for x in payload)


# ---------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    cfg = si.CONFIGS[args.config]
    tau = args.tau if args.tau is not None else cfg.tau
    iters = args.iters if args.iters is not None else cfg.iters
    kind, payload = si.make_input(cfg)
    config = run_config(args, cfg, ws, payload_bytes(kind, payload))
    import oracle as O
    if kind == "dense":
        So = O.OMat.from_dense(payload, cfg.b)
    else:
        So = O.OMat.from_blocks(cfg.n, cfg.b, *payload)
    # c from the oracle's own power iteration, once (not part of the timed samples)
    c = O.power_scale(So, 100)
    del So
    for _ in range(args.warmup):
        oracle_sample(cfg, payload, tau, args.ref_iters, c, tau * cfg.tau_s_factor)
    tot_t, tot_f, cores, per_k, build_s = 0.0, 0.0, 1, [], []
    for _ in range(args.steps):
        dt, fl, cores, pk, bs = oracle_sample(cfg, payload, tau, args.ref_iters, c, tau * cfg.tau_s_factor)
        tot_t += dt
        tot_f += fl
        per_k.append(pk)
        build_s.append(bs)
    value = tot_f / tot_t / 1e12
    sample = (f"{args.config} input, oracle quadtree build + Y0 + the first {args.ref_iters} of "
              f"{iters} NS iterations per step (c given)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model(), "s_per_k": [statistics.mean(x) for x in zip(*per_k)],
                         "build_s": statistics.mean(build_s)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import paper_1508_05856_b200 as sp
    from paper_1508_05856_b200 import dist as D

    ws, rank, local = dist_env()
    dist = None
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if ws > 1 or args.dist_world1:
        import torch.distributed as dist
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    cfg = si.CONFIGS[args.config]
    tau = args.tau if args.tau is not None else cfg.tau
    iters = args.iters if args.iters is not None else cfg.iters
    tau_s = tau * (args.tau_s_factor if args.tau_s_factor is not None else cfg.tau_s_factor)
    t_stop = args.t_stop if args.t_stop is not None else cfg.t_stop
    scaled = args.map == "scaled"
    nb = cfg.n // cfg.b

    # ---- row partition over the ranks; fixed for the run
    comm, row_start, rows = None, None, (0, nb)
    if dist is not None:
        comm = D.init_nccl_comm(local)
        if args.partition == "balanced":
            # per-row leaf task counts of s (x)_tau s from the replicated norms (setup, untimed)
            kind, full = si.make_input(cfg)
            c0 = sp.spamm_ctx_create(local)
            S0 = (sp.spamm_build_tree(c0, torch.from_numpy(full).to(dev), cfg.b) if kind == "dense" else
                  sp.spamm_build_tree_blocks(c0, cfg.n, cfg.b, *(torch.from_numpy(x).to(dev) for x in full)))
            row_start = D.balanced_partition(sp.spamm_row_task_counts(c0, S0, S0, tau), ws)
            S0.free()
            c0.close()
            del full
        else:
            row_start = D.equal_partition(nb, ws)
        rows = (row_start[rank], row_start[rank + 1])
    kind, payload = si.make_input(cfg, rows=rows if comm is not None else None)
    ctx = sp.spamm_ctx_create(local, torch_allocator=args.allocator == "torch")
    if comm is not None:
        sp.spamm_ctx_set_comm(ctx, comm, row_start)
    stream = ctx.stream

    if kind == "dense":
        d_in = (torch.from_numpy(payload).to(dev),)
        h_in = (torch.from_numpy(payload).pin_memory(),)
        in_bytes = payload.nbytes
    else:
        bi, bj, blocks = payload
        d_in = tuple(torch.from_numpy(x).to(dev) for x in (bi, bj, blocks))
        h_in = tuple(torch.from_numpy(x).pin_memory() for x in (bi, bj, blocks))
        in_bytes = bi.nbytes + bj.nbytes + blocks.nbytes

    def build(inp):
        if kind == "dense":
            return sp.spamm_build_tree(ctx, inp[0], cfg.b)
        return sp.spamm_build_tree_blocks(ctx, cfg.n, cfg.b, *inp)

    out_host = {}

    def step(inp, readback):
        S = build(inp)
        if args.channel == "single":
            r = sp.spamm_ns_sqrt_single(ctx, S, tau, iters, tau_s=tau_s, t_stop=t_stop, scaled=scaled)
        else:
            r = sp.spamm_ns_sqrt(ctx, S, tau, iters, tau_s=tau_s, mu=cfg.mu, t_stop=t_stop, scaled=scaled)
        S.free()
        flops = sum(p["flops"] for k in r["stats"] for p in k)
        tasks = sum(p["tasks"] for k in r["stats"] for p in k)
        d2h = 0
        if readback:
            for key in ("Y", "Z"):
                nblk = r[key].nblocks
                buf = out_host.get(key)
                if buf is None or buf[0].shape[0] < nblk:
                    cap = int(nblk * 1.25) + 16
                    buf = (torch.empty(cap, dtype=torch.int32).pin_memory(),
                           torch.empty(cap, dtype=torch.int32).pin_memory(),
                           torch.empty((cap, cfg.b, cfg.b), dtype=torch.float64).pin_memory())
                    out_host[key] = buf
                sp.spamm_export_blocks(ctx, r[key], buf)
                d2h += nblk * (8 + 8 * cfg.b * cfg.b)
        r["Y"].free()
        r["Z"].free()
        return flops, tasks, d2h, r

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- FP64 tensor peak on this GPU (DMMA issue-rate microbenchmark, ~2 s sustained)
    _, ms1 = sp.spamm_peak_dmma(ctx, 20000)
    peak_tflops, peak_ms = sp.spamm_peak_dmma(ctx, int(20000 * max(1.0, 2000.0 / max(ms1, 1e-3))))
    # cross-check of the denominator: a library FP64 GEMM (cuBLAS DGEMM via torch.matmul),
    # 8192^3, best of 5 (context only; not used in any ratio)
    dgemm_tflops = None
    try:
        ga = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
        gb = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
        torch.matmul(ga, gb)
        best = 1e30
        for _ in range(5):
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            torch.matmul(ga, gb)
            g1.record()
            torch.cuda.synchronize()
            best = min(best, g0.elapsed_time(g1))
        dgemm_tflops = 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12
        del ga, gb
        torch.cuda.empty_cache()
    except RuntimeError:
        pass

    # ---- warm-up
    for _ in range(args.warmup):
        step(d_in, False)
    torch.cuda.synchronize()

    # ---- timed: inputs resident in HBM (s: block list > L2)
    clocks = Clocks(local)
    sp.spamm_profile_enable(ctx, True)
    l0 = sp.spamm_kernel_launches(ctx)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    flops = tasks = 0.0
    last = None
    for _ in range(args.steps):
        f, t, _, last = step(d_in, False)
        flops += f
        tasks += t
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = sp.spamm_kernel_launches(ctx) - l0
    prof = sp.spamm_profile_read(ctx)
    sp.spamm_profile_enable(ctx, False)
    ms_max = D.max_over_ranks(ms, dev)
    flops_all = D.sum_over_ranks(flops, dev)
    tasks_all = D.sum_over_ranks(tasks, dev)
    value = flops_all / (ms_max * 1e-3) / 1e12
    rank_tasks = D.gather_to_rank0(tasks / args.steps)

    # ---- roofline of the dominant kernel (leaf GEMM), algorithmic flops / event time
    gemm_achieved = prof["gemm_flops"] / (prof["gemm_ms"] * 1e-3) / 1e12 if prof["gemm_ms"] else None
    roofline = {
        "bound": "tensor", "achieved": gemm_achieved, "peak": peak_tflops, "unit": "TFLOP/s",
        "frac": (gemm_achieved / peak_tflops) if gemm_achieved else None, "traffic": None,
        "kernel": "k_leaf_gemm (FP64 DMMA m8n8k4)",
        "cublas_dgemm_8192_tflops": dgemm_tflops,
        "peak_source": "measured in this run: spamm_peak_dmma (back-to-back DMMA on all SMs, "
                       f"{peak_ms:.0f} ms); MEASURED_PEAKS.json has no FP64 figure",
        "launches": prof["gemm_count"], "avg_launch_ms": prof["gemm_ms"] / max(prof["gemm_count"], 1),
        "gemm_share_of_step": prof["gemm_ms"] / ms if ms else None,
        "flops_per_launch": prof["gemm_flops"] / max(prof["gemm_count"], 1),
    }
    traffic_file = os.path.join(ROOT, "profiles", f"gemm_traffic_{args.config}.json")
    if os.path.exists(traffic_file):
        try:
            tf = json.load(open(traffic_file))
            roofline["traffic"] = tf.get("bytes_per_launch")
            roofline["traffic_source"] = tf.get("source")
        except (OSError, ValueError):
            pass

    # ---- e2e through the C ABI with HOST buffers: every step passes its input as pinned
    # HOST pointers to spamm_build_tree[_blocks] (the library stages it to the device on
    # its stream: H2D inside the step) and reads Y and Z back into pinned HOST buffers with
    # spamm_export_blocks_async (the library's copy stream: each step's D2H overlaps the
    # next step's compute); spamm_copies_join puts the last copies inside the timed region.
    e2e = None
    if not args.no_e2e:
        hout = [{}, {}]

        def hbufs(i, key, nblk):
            h = hout[i].get(key)
            if h is None or h[0].shape[0] < nblk:
                cap = int(nblk * 1.25) + 16
                h = hout[i][key] = (torch.empty(cap, dtype=torch.int32).pin_memory(),
                                    torch.empty(cap, dtype=torch.int32).pin_memory(),
                                    torch.empty((cap, cfg.b, cfg.b), dtype=torch.float64).pin_memory())
            return h

        def upload():
            # the library's asynchronous upload (prefetch half of the build)
            if kind == "dense":
                return sp.spamm_stage_dense(ctx, h_in[0])
            return sp.spamm_stage_blocks(ctx, cfg.b, *h_in)

        def e2e_step(i, staged, last):
            S = sp.spamm_build_tree_staged(ctx, cfg.n, cfg.b, staged)   # waits for its H2D
            nxt = None if last else upload()          # next input's H2D overlaps this step
            if args.channel == "single":
                r = sp.spamm_ns_sqrt_single(ctx, S, tau, iters, tau_s=tau_s, t_stop=t_stop, scaled=scaled)
            else:
                r = sp.spamm_ns_sqrt(ctx, S, tau, iters, tau_s=tau_s, mu=cfg.mu, t_stop=t_stop, scaled=scaled)
            S.free()
            nbytes = 0
            for key in ("Y", "Z"):
                nblk = sp.spamm_export_blocks_async(ctx, r[key], hbufs(i % 2, key, r[key].nblocks))
                nbytes += nblk * (8 + 8 * cfg.b * cfg.b)
                r[key].free()
            flops = sum(p["flops"] for k in r["stats"] for p in k)
            return flops, nbytes, nxt

        st_ = upload()
        for i in range(2):                            # allocate the buffers (untimed)
            _, _, st_ = e2e_step(i, st_, last=i == 1)
        sp.spamm_copies_wait(ctx)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        ef = 0.0
        d2h = 0
        st_ = upload()
        for i in range(args.steps):
            f, d2h, st_ = e2e_step(i, st_, last=i == args.steps - 1)
            ef += f
        sp.spamm_copies_join(ctx)
        e3.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = D.max_over_ranks(e2.elapsed_time(e3), dev)
        e2e = {"value": D.sum_over_ranks(ef, dev) / (ems * 1e-3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": int(D.sum_over_ranks(in_bytes, dev)),
               "d2h_bytes_per_step": int(D.sum_over_ranks(d2h, dev)),
               "ms_per_step": ems / args.steps,
               "path": "C ABI host pointers: spamm_stage_blocks / spamm_stage_dense (pinned host input; H2D "
                       "on the library's upload stream, issued for step i+1 while step i computes) + "
                       "spamm_build_tree_staged; spamm_export_blocks_async "
                       "(pinned host output; D2H on the library's copy stream, overlapping the next step) "
                       "+ spamm_copies_join"}

    # ---- seconds per NS iteration k (BJ:2), from one extra untimed run driven step by
    # step (spamm_ns_step, CUDA events on the library stream around each k)
    per_k = None
    if args.channel == "dual" and not scaled:
        S = build(d_in)
        c = sp.spamm_power_scale(ctx, S, 100)
        Y, Z = sp.spamm_ns_y0(ctx, S, c, cfg.mu), sp.spamm_identity(ctx, cfg.n, cfg.b)
        S.free()
        per_k = []
        for _ in range(iters):
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(stream)
            Yn, Zn, t, _ = sp.spamm_ns_step(ctx, Y, Z, tau, tau_s)
            k1.record(stream)
            k1.synchronize()
            per_k.append(k0.elapsed_time(k1) / 1e3)
            Y.free()
            Z.free()
            Y, Z = Yn, Zn
            if t_stop > 0 and abs(t) <= t_stop:
                break
        Y.free()
        Z.free()

    # ---- BASELINE.json's literal configuration (tau_s = tau, the config's fixed iteration
    # count, no convergence exit), when the bench workload re-scopes it (readings L9/L15):
    # one untimed run, its outcome recorded
    literal = None
    if args.channel == "dual" and not scaled and (tau_s != tau or t_stop > 0):
        S = build(d_in)
        t0 = time.perf_counter()
        r = sp.spamm_ns_sqrt(ctx, S, tau, iters, tau_s=tau, mu=cfg.mu, check=False)
        dt = time.perf_counter() - t0
        S.free()
        if "status" in r:
            literal = {"tau_s": tau, "iters": iters, "t_stop": 0.0,
                       "outcome": f"diverges: {r['error']} after {r['iters']} completed steps",
                       "t_history": [float(x) for x in r["t"]], "wall_s": dt,
                       "oracle": "tests/test_gpu_fullsize.py::test_c5_tau_s_equal_tau_divergence_is_the_methods "
                                 "(the oracle's step from the GPU's Y_9, Z_9 reproduces ||Z|| x2.37 and t_10 = 2.5598)"}
        else:
            literal = {"tau_s": tau, "iters": iters, "t_stop": 0.0, "outcome": "completed",
                       "t_final": float(r["t"][-1]), "wall_s": dt,
                       "tasks": int(sum(p["tasks"] for k in r["stats"] for p in k))}
            r["Y"].free()
            r["Z"].free()

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        S = build(d_in)
        c = sp.spamm_power_scale(ctx, S, 100)
        S.free()
        dt, fl, cores, cpu_per_k, build_s = oracle_sample(cfg, payload, tau, args.ref_iters, c, tau_s)
        cpu = {"value": fl / dt / 1e12, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{args.config} input: oracle quadtree build + Y0 + first {args.ref_iters} "
                         f"of {iters} NS iterations ({fl:.3g} culled-leaf flop in {dt:.1f} s)",
               "cpu": cpu_model(), "s_per_k": cpu_per_k, "build_s": build_s}

    blocks_mb = D.sum_over_ranks(in_bytes, dev) / 1e6
    if rank == 0:
        r = last
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": run_config(args, cfg, ws, blocks_mb * 1e6),
            "iters_run": int(r["iters"]),
            "s_per_ns_iteration": prof["loop_ms"] / args.steps / max(int(r["iters"]), 1) / 1e3,
            "s_per_k": per_k,
            "s_per_k_source": "one extra untimed run driven by spamm_ns_step (host-driven, no graph/"
                              "chaining), CUDA events around each k",
            "setup_ms_per_step": prof["setup_ms"] / args.steps,
            "tasks_per_step": tasks_all / args.steps,
            "t_final": float(r["t"][-1]) if len(r["t"]) else None,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "baseline_literal": literal,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "phase_ms_per_step": {k: prof[f"{k}_ms"] / args.steps
                                  for k in ("gemm", "cull", "setup", "loop", "other")},
        }
        if comm is not None:
            line["partition"] = {"row_start": row_start, "tasks_per_rank": rank_tasks,
                                 "imbalance": max(rank_tasks) / (sum(rank_tasks) / ws)}
        print(json.dumps(line), flush=True)
    if comm is not None:
        ctx.close()
        comm.destroy()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def watchdog(seconds: float):
    """A multi-rank run whose peer died would wait in a collective forever: after `seconds`
    this rank reports and exits non-zero instead (SPAMM_BENCH_TIMEOUT, default 1 h; 0 = off)."""
    if seconds <= 0:
        return
    import threading

    def fire():
        ws, rank, _ = dist_env()
        print(json.dumps({"error": f"bench.py watchdog: rank {rank}/{ws} still running after {seconds:.0f} s"}),
              file=sys.stderr, flush=True)
        os._exit(3)
    t = threading.Timer(seconds, fire)
    t.daemon = True
    t.start()


def main():
    args = parse()
    watchdog(float(os.environ.get("SPAMM_BENCH_TIMEOUT", "3600")))
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
