"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
markdown table: launches and microseconds per training step (steps = adamw
launches), share of the summed kernel time.  usage: python tools/launch_summary.py CSV"""
import collections
import csv
import re
import sys


def short(name):
    m = re.search(r"(TcRow|TcRed|RedStore|ChunkStore|EmbedStore)<[^<>]*?(\w+Prob|\w+Grad|\w+Dh)?>", name)
    base = re.search(r"(\w+)(?:<|\()", name)
    k = base.group(1) if base else name[:40]
    if "chain_kernel" in name or "pair_kernel" in name:
        t = re.search(r"(chain|pair)_kernel<([^>]*)>", name)
        return f"{t.group(1)}<{t.group(2)}>" if t else k
    p = re.search(r"::(\w+(?:Prob|Grad|Dh))>", name)
    return f"{k}<{p.group(1)}>" if p else k


lines = open(sys.argv[1]).read().splitlines()
lines = lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]  # (ncu log lines before the header)
rows = list(csv.DictReader(lines))
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1000.0 if r["Metric Unit"] in ("nsecond", "ns") else v * (1000.0 if r["Metric Unit"] in ("msecond", "ms") else 1.0)
    k = short(r["Kernel Name"])
    tot[k][0] += 1
    tot[k][1] += us
steps = max(1, tot.get("adamw_kernel", [1])[0])
total = sum(v[1] for v in tot.values())
print(f"# {sum(v[0] for v in tot.values())} launches, {steps} training steps, {total / steps:.1f} us of kernel time per step "
      "(ncu, serialised, cold L2 per kernel; shares, not absolute step time)\n")
print("| kernel | launches / step | us / step | us / launch | share |")
print("|---|---:|---:|---:|---:|")
for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:45]:
    print(f"| `{k}` | {n / steps:.1f} | {us / steps:.1f} | {us / n:.1f} | {us / total:.3f} |")
