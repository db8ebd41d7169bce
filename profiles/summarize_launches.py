"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.

usage: python profiles/summarize_launches.py <launches.csv> [--last-step]
With --last-step, only the final repetition of the step's launch sequence (a
graph replay) is summarised.  ncu serialises kernels (no stream overlap), so
the sum exceeds the step time; compare SHARES.
"""
import csv
import re
import sys
from collections import defaultdict


def short(n):
    m = re.search(r"split_reduce_kernel<.*?(ChunkStore|EmbedStore|RedStore)", n)
    if m:
        return "split_reduce<" + m.group(1) + ">"
    m = re.search(r"(TcRow|TcRed)<.*?::(\w+Prob|\w+Grad|F0Dh)>", n)
    if m:
        return f"{'tc_row' if m.group(1) == 'TcRow' else 'tc_red'}<{m.group(2)}>"
    m = re.search(r"chain_kernel<(\d+), (\d+), \(?(?:int\))?(-?\d+)(?:, \d+)?>", n)
    if m:
        return "chain<%s,%s,%s>" % m.groups()
    m = re.search(r"(gemm_ab_kernel|gemm_atb_kernel|gemm_atb_reduce|bimg_prob_kernel)<[^>]*?(\w+Prob|\w+Grad|F0Dh)\b", n)
    if m:
        return f"{m.group(1)}<{m.group(2)}>"
    m = re.search(r"(\w+)\(", n)
    return m.group(1) if m else n[:60]


def main():
    rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    if "--last-step" in sys.argv:
        names = [r["Kernel Name"] for r in rows]
        for k in range(20, len(names) // 2 + 1):
            if names[-k:] == names[-2 * k:-k]:
                rows = rows[-k:]
                break
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        a = agg[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", "")) / 1e3
    total = sum(v[1] for v in agg.values())
    print(f"# {len(rows)} launches, {total:.1f} us of kernel time (ncu, serialised)\n")
    print("| kernel | launches | total us | us / launch | share |\n|---|---:|---:|---:|---:|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {us:.1f} | {us / n:.1f} | {us / total:.3f} |")


if __name__ == "__main__":
    main()
