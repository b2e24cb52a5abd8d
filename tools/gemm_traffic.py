"""profiles/gemm_traffic_<cfg>.json (bench.py's roofline.traffic source) and the key-counter
summary of an ncu --set full capture of the three leaf-GEMM launches (X, Y', Z') of one NS
iteration, run here after gpurun:

  gpurun: ncu --set full --clock-control none -k regex:k_leaf_gemm -s 3k -c 3 -o rep \
              python tools/diag_ns.py --config C5 --iters k+1 --tau-s 1e-9 > diag.log
  here:   python tools/gemm_traffic.py C5 rep.ncu-rep diag.log k "<the ncu command>"
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import report  # noqa: E402

cfg, rep, log, k, cmd = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5]
b = 64
tasks = None
for line in open(log):
    m = re.match(r"k=\s*(\d+) .*tasks=\[(\d+), (\d+), (\d+)\]", line)
    if m and int(m.group(1)) == k:
        tasks = [int(m.group(i)) for i in (2, 3, 4)]
assert tasks, f"iteration {k} not in {log}"
r = report(rep)
assert len(r) == 3, len(r)
unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "msecond": 1e-3,
        "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9, "%": 1.0, "cycle": 1.0}


def val(e, key):
    v, u = e[key]
    return float(v.replace(",", "")) * unit.get(u, 1.0)


launches = []
for e, t in zip(r, tasks):
    f = 2.0 * b ** 3 * t
    ts = val(e, "gpu__time_duration.sum")
    rd, wr = val(e, "dram__bytes_read.sum"), val(e, "dram__bytes_write.sum")
    launches.append(dict(kernel=e["kernel"], tasks=t, flops=f, time_s=ts, tflops=f / ts / 1e12,
                         dram_read=rd, dram_write=wr, dram_total=rd + wr,
                         dmma_active_frac=val(e, "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg")
                         / val(e, "sm__cycles_elapsed.avg"),
                         l2_hit_pct=val(e, "lts__t_sector_hit_rate.pct"),
                         operand_bytes_if_no_reuse=2 * 8 * b * b * t))
out = dict(kernel=f"k_leaf_gemm<64,...> ({cfg}, NS iteration k={k}: X, Y', Z' launches)",
           bytes_per_launch=sum(x["dram_total"] for x in launches) / 3,
           flops_per_launch=sum(x["flops"] for x in launches) / 3,
           source=cmd, launches=launches,
           note="dram write = the output blocks; dram read = the unique operand blocks plus what L2 "
                "(126 MB) cannot hold of the operand stream (C3: ~compulsory; C5 Y': ~1.8x the "
                "unique blocks, DESIGN.md section 5)")
json.dump(out, open(os.path.join("profiles", f"gemm_traffic_{cfg}.json"), "w"), indent=1)
json.dump(r, open(os.path.join("profiles", os.environ.get("SPAMM_ROUND", "r02"), f"gemm_{cfg}_k{k}_full.json"), "w"), indent=1)
for x in launches:
    print(f"{x['kernel'][:48]:48s} tasks {x['tasks']:8d} {x['time_s'] * 1e3:8.3f} ms {x['tflops']:6.2f} TF "
          f"DMMA active {x['dmma_active_frac']:.3f} DRAM {x['dram_total'] / 1e9:6.2f} GB L2 hit {x['l2_hit_pct']:.1f}%")
