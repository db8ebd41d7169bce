# GPU suite + default bench (no CPU baseline) + per-kernel table
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print(d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], "launches/step", d["gpu_launches"] / d["steps"])
for k, v in list(d["kernel_ms_per_step"].items())[:22]:
    print(f"{k:32s} {v:8.4f} {d['kernel_launches_per_step'][k]}")
PY
