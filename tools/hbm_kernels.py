"""ncu --set full summary of the HBM / latency-bound kernels (norm build, pyramid, cull,
maps, SpMV): achieved DRAM GB/s against the measured copy bandwidth (MEASURED_PEAKS.json)."""
import json
import subprocess
import sys

rep = sys.argv[1]
peak = 6535.4
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
import csv  # noqa: E402
rows = list(csv.reader(raw.splitlines()))
h, units, data = rows[0], rows[1], rows[2:]


def get(row, key):
    i = h.index(key)
    v = float(row[i].replace(",", ""))
    u = units[i]
    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}.get(u, 1.0)


out = []
for row in data:
    name = row[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    t = get(row, "gpu__time_duration.sum")
    rd, wr = get(row, "dram__bytes_read.sum"), get(row, "dram__bytes_write.sum")
    out.append(dict(kernel=name, time_us=t * 1e6, dram_read_MB=rd / 1e6, dram_write_MB=wr / 1e6,
                    achieved_GBs=(rd + wr) / t / 1e9, frac_of_copy_bw=(rd + wr) / t / 1e9 / peak,
                    grid=row[h.index("launch__grid_size")], regs=row[h.index("launch__registers_per_thread")]))
for o in out:
    print(f"{o['kernel']:28s} {o['time_us']:8.1f} us  R {o['dram_read_MB']:8.1f} MB  W {o['dram_write_MB']:8.1f} MB"
          f"  {o['achieved_GBs']:7.0f} GB/s  ({100 * o['frac_of_copy_bw']:.0f}% of {peak:.0f})")
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
