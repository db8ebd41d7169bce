mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity_measured.py -x -q > gpurun_out/fused.log 2>&1; echo "tests rc=$?" >> gpurun_out/fused.log
HMTL_BENCH_NAMES=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; echo bench rc=$?
NCU_SPECS="msgseg|tc_row_kernel.*MsgSegProb|0 l7seg|tc_row_kernel.*L7SegProb|0 segsrc|seg_src_kernel|0" bash tools/gpu/ncu_fused.sh
tail -3 gpurun_out/fused.log
