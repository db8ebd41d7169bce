"""Key metrics of `ncu --page raw --csv` exports.  usage: python tools/ncu_summary.py a.raw.csv ..."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "dur"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("lts__t_bytes.sum", "l2_bytes"), ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("lts__t_sector_hit_rate.pct", "l2hit%"),
        ("sm__cycles_active.avg", "sm_active_cyc"), ("gpc__cycles_elapsed.max", "elapsed_cyc"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%")]
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        print(f, "empty")
        continue
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    print(f.split("/")[-1], d.get("Kernel Name", "")[:60])
    print("   " + "  ".join(f"{n}={d[k]}{u[k] if u[k] not in ('', '%') else ''}" for k, n in KEYS if k in d))
