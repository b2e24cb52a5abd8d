"""Print the DESIGN.md measurement-table rows from a directory of bench lines
(profiles/r02/<run>/bench_*.json):  python tools/bench_table.py profiles/r02/final6"""
import glob
import json
import os
import sys

d = sys.argv[1]
print("| file | iterations | tasks / run | ms / run (setup, loop) | culled-leaf TFLOP/s | e2e TFLOP/s | GEMM frac | SM MHz, reasons |")
print("|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
    try:
        x = json.loads(open(f).read().strip().splitlines()[-1])
    except (IndexError, ValueError):
        print(f"| {os.path.basename(f)} | unreadable |")
        continue
    if x.get("impl") == "reference":
        print(f"| {os.path.basename(f)} | reference arm (CPU oracle, {x['cpu_baseline']['cores']} cores): "
              f"{x['value']:.4f} {x['unit']}, {x['ms_per_step']:.0f} ms per sampled step |")
        continue
    ph = x.get("phase_ms_per_step", {})
    e = x.get("e2e") or {}
    print(f"| {os.path.basename(f)} | {x.get('iters_run')} | {x.get('tasks_per_step', 0):.3g} | "
          f"{x['ms_per_step']:.2f} ({ph.get('setup', 0):.2f}, {ph.get('loop', 0):.2f}) | {x['value']:.4g} | "
          f"{e.get('value', float('nan')):.4g} | {x['roofline']['frac']:.3f} | "
          f"{x['clocks']['sm_mhz']:.0f}, {x['clocks']['reasons']} |")
