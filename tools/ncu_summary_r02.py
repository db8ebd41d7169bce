"""Summarise ncu --set full raw CSVs (one kernel each) into a markdown table:
duration, DRAM bytes and bandwidth, tensor-pipe utilisation, warps active, registers.
python tools/ncu_summary_r02.py gpurun_out/ncu/<name>.raw.csv ... > profiles/r02/ncu_summary.md"""
import csv
import os
import sys

SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
TSCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def one(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    f = lambda k: float(d[k].replace(",", "")) if d.get(k) not in (None, "", "n/a") else float("nan")
    t = f("gpu__time_duration.sum") * TSCALE.get(u.get("gpu__time_duration.sum", "us"), 1.0)
    mb = f("dram__bytes_read.sum") * SCALE.get(u.get("dram__bytes_read.sum"), 1.0) + \
        f("dram__bytes_write.sum") * SCALE.get(u.get("dram__bytes_write.sum"), 1.0)
    return {"kernel": d.get("Kernel Name", "")[:70], "us": t, "dram_MB": mb, "TBps": mb / t if t else 0.0,
            "tensor": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            "tc": f("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"),
            "warps": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": d.get("launch__registers_per_thread", ""), "grid": d.get("launch__grid_size", "")}


print("| capture | kernel | us (cold) | DRAM MB | DRAM TB/s | tensor pipe % | tc pipe % | warps active % | regs | grid |")
print("|---|---|---:|---:|---:|---:|---:|---:|---:|---:|")
for p in sys.argv[1:]:
    r = one(p)
    if r:
        print(f"| {os.path.basename(p).split('.')[0]} | `{r['kernel']}` | {r['us']:.1f} | {r['dram_MB']:.1f} | "
              f"{r['TBps']:.2f} | {r['tensor']:.1f} | {r['tc']:.1f} | {r['warps']:.1f} | {r['regs']} | {r['grid']} |")
