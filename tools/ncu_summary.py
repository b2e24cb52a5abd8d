"""Summarise ncu outputs into profiles/ (run here, on the CPU side, after gpurun).

  python tools/ncu_summary.py launches <launches.csv>           per-kernel share of device time
  python tools/ncu_summary.py report <x.ncu-rep> [--json out]   key counters of a --set full capture
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    r = csv.reader(lines)
    hdr = next(r)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for row in r:
        name = row[ki].split("(")[0].replace("void ", "").split("<")[0].strip()
        v = float(row[vi].replace(",", "")) * scale.get(row[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    # the library's kernels only: the DMMA peak probe and the cuBLAS DGEMM cross-check that
    # bench.py runs before the timed region are not part of the path
    def ours(k):
        return k.startswith("k_") and k != "k_peak_dmma"
    tot = sum(v[1] for k, v in agg.items() if ours(k))
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        if not ours(k):
            continue
        out.append(f"{k:28s} launches {v[0]:6d}  total {v[1] / 1e3:10.3f} ms  avg {v[1] / v[0]:9.2f} us  "
                   f"share {100 * v[1] / tot:6.2f}%")
    out.append(f"total (library kernels; excluding the DMMA peak probe and the cuBLAS cross-check) {tot / 1e3:.3f} ms")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
        "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "gpc__cycles_elapsed.avg.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        e = {"kernel": d[hdr.index("Kernel Name")][:80]}
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k or h.endswith("." + k) or h.endswith(k):
                    if h.split(".")[-1] != k.split(".")[-1]:
                        continue
                    e[k] = (d[i], units[i])
                    break
        res.append(e)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        r = report(sys.argv[2])
        print(json.dumps(r, indent=1))
