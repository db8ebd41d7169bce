"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

usage: python profiles/summarize_launches.py <launches.csv> [--steps S]
Per-launch ncu times are cold-cache and serialised: compare SHARES, not absolutes.
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    m = re.search(r"(gemm_ab_kernel|gemm_atb_kernel|gemm_atb_reduce)<[^>]*?(\w+Prob|\w+Grad|F0Dh)\b", name)
    if m:
        return f"{m.group(1)}<{m.group(2)}>"
    m = re.search(r"::(\w+)\(", name)
    return m.group(1) if m else name[:60]


def main():
    path = sys.argv[1]
    steps = float(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1.0
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"].replace(",", ""))
    total = sum(v[1] for v in agg.values())
    print(f"# {len(rows)} launches, {total / 1e6:.3f} ms total (ncu, serialised, cold cache)\n")
    print("| kernel | launches | total us | share |")
    print("|---|---:|---:|---:|")
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {ns / 1e3:.1f} | {ns / total:.3f} |")


if __name__ == "__main__":
    main()
