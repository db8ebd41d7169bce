# round 2: measured-config parity tests + bench lines for every workload
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity_measured.py -x -q -s > gpurun_out/parity_measured.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity_measured.log
timeout 900 python bench.py > gpurun_out/bench_mtl5.json 2> gpurun_out/bench_mtl5.err; echo "mtl5 rc=$?"
timeout 900 python bench.py --workload cfg2 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --workload cfg4 --cpu-seconds 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_mtl5.json 2> gpurun_out/bench_ref_mtl5.err; echo "ref rc=$?"
tail -3 gpurun_out/parity_measured.log
