mkdir -p gpurun_out
python tools/mma_rate.py 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python tools/tc_bench.py 2>&1 | tail -20
bash tools/gpu/bench_quick.sh 2>&1 | head -3
