"""Kernel timeline of one graph step (torch.profiler / CUPTI): start, duration and
stream of every kernel, per-stream busy time, and the main-stream gaps.
python tools/timeline.py [--json out.json]"""
import ctypes as C, json, os, re, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import torch
import bench
import paper_2506_21788_b200 as P
from paper_2506_21788_b200._lib import check, lib


def short(n):
    for pat, fmt in ((r"(TcRow|TcRed)<.*?::(\w+Prob|\w+Grad|F0Dh)>", "{0}<{1}>"), (r"chain_kernel<(\d+), (\d+), \(?(?:int\))?(-?\d+)(?:, \d+)?>", "chain<{0},{1},{2}>"),
                     (r"split_reduce_kernel<.*?(ChunkStore|EmbedStore|RedStore)", "split<{0}>")):
        m = re.search(pat, n)
        if m:
            return fmt.format(*m.groups())
    m = re.search(r"(\w+)\(", n)
    return m.group(1) if m else n[:40]


heads, batches, _ = bench.rank_batches(0, 1)
caps = P.Caps.for_samples(batches[0])
for b in batches[1:]:
    caps = caps.union(P.Caps.for_samples(b))
m = P.ModelT(P.ModelHyper(**bench.HYPER), 7, heads, caps=caps)
slots = []
for b in batches:
    sl = C.c_int()
    check(lib().hmtl_pool_add(m.ctx, C.byref(b.as_c()), C.byref(sl)))
    slots.append(sl.value)
cfg = P.TrainConfig(use_graph=True)
for i in range(6):
    check(lib().hmtl_pool_bind(m.ctx, slots[i % 4], None))
    check(lib().hmtl_train_step(m.ctx, C.byref(cfg.c()), None))
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA], acc_events=True) as prof:
    for i in range(3):
        check(lib().hmtl_pool_bind(m.ctx, slots[i % 4], None))
        check(lib().hmtl_train_step(m.ctx, C.byref(cfg.c()), None))
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
# the last step: from the last adamw-preceding prep_kernel
starts = [i for i, e in enumerate(ev) if short(e["name"]) == "prep_kernel"]
step = ev[starts[-1]:]
t0 = step[0]["ts"]
end = max(e["ts"] + e["dur"] for e in step)
print(f"step span {end - t0:.1f} us, {len(step)} kernels")
busy = {}
for e in step:
    s = e["args"].get("stream", 0)
    busy[s] = busy.get(s, 0) + e["dur"]
print("busy per stream (us):", {k: round(v, 1) for k, v in busy.items()})
main = max(busy, key=busy.get)
prev = t0
gaps = 0.0
rows = []
for e in step:
    s = e["args"].get("stream", 0)
    if s == main:
        gaps += max(0.0, e["ts"] - prev)
        prev = max(prev, e["ts"] + e["dur"])
    rows.append((e["ts"] - t0, e["dur"], s, short(e["name"])))
print(f"main stream {main}: idle gaps {gaps:.1f} us")
for r in rows:
    print(f"{r[0]:8.1f} {r[1]:7.1f}  s{r[2]:<4} {r[3]}")
if "--json" in sys.argv:
    json.dump(rows, open(sys.argv[sys.argv.index("--json") + 1], "w"))
