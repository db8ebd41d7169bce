# quick 1-GPU bench (no CPU baseline) -> gpurun_out/bq.json
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bq.json 2> gpurun_out/bq.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bq.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"], "launches", d["gpu_launches"])
print("roofline", d["roofline"])
print("gs", d["roofline_gather_scatter"])
tot = sum(d["kernel_ms_per_step"].values())
print("sum of scopes ms", round(tot, 4))
for k, v in d["kernel_ms_per_step"].items():
    print(f"  {k:28s} {v:.4f}")
PY
