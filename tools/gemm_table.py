"""Per-GEMM table from an ncu metrics CSV (tools/gpu/ncu_gemms.sh): the last graph
step's instance of every tensor-core GEMM kernel -- duration (cold L2), tensor-pipe
utilisation, DRAM bytes, warps active, grid.  usage: python tools/gemm_table.py CSV"""
import collections
import csv
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
lines = lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]
rows = list(csv.DictReader(lines))
by_id = collections.OrderedDict()
for r in rows:
    d = by_id.setdefault(r["ID"], {"name": r["Kernel Name"]})
    v = r["Metric Value"].replace(",", "")
    u = r["Metric Unit"]
    try:
        x = float(v)
    except ValueError:
        continue
    if r["Metric Name"] == "gpu__time_duration.sum":
        x = x / 1000.0 if u in ("nsecond", "ns") else x * (1000.0 if u in ("msecond", "ms") else 1.0)
    if r["Metric Name"].startswith("dram__bytes"):
        x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
    d[r["Metric Name"]] = x


def short(n):
    t = re.search(r"(chain_kernel<[^>]*>)", n)
    if t:
        return t.group(1)
    p = re.search(r"::(\w+(?:Prob|Grad|Dh))>", n)
    k = re.search(r"(tc_row_kernel|tc_red_tma_kernel|tc_red_kernel)", n)
    return f"{k.group(1) if k else n[:30]}<{p.group(1) if p else '?'}>"


last = collections.OrderedDict()
for i, d in by_id.items():
    last.setdefault(short(d["name"]), []).append(d)
print("| GEMM kernel | instances (3 steps) | us (cold, last) | tensor pipe % | tc pipe % | DRAM MB | warps active % | grid |")
print("|---|---:|---:|---:|---:|---:|---:|---:|")
for k, ds in last.items():
    d = ds[-1]
    g = lambda m: d.get(m, float("nan"))
    print(f"| `{k}` | {len(ds)} | {g('gpu__time_duration.sum'):.1f} | {g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g('sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{g('dram__bytes_read.sum') + g('dram__bytes_write.sum'):.1f} | {g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | {g('launch__grid_size'):.0f} |")
