# round-2 final numbers on the final build: bench lines (mtl5 with cpu_baseline, cfg2,
# cfg4, reference arm) + the measured-configuration parity log
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests/test_gpu_parity_measured.py -q -s > gpurun_out/final/parity_measured.log 2>&1; echo "parity rc=$?"
timeout 900 python bench.py > gpurun_out/final/bench_mtl5.json 2> gpurun_out/final/bench_mtl5.err; echo "mtl5 rc=$?"
timeout 900 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --workload cfg4 --no-cpu-baseline > gpurun_out/final/bench_cfg4.json 2> gpurun_out/final/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo "ref rc=$?"
for f in mtl5 cfg2 cfg4 reference; do python -c "import json;d=json.loads(open('gpurun_out/final/bench_$f.json').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('parity') or {}), d.get('clocks'))" 2>&1 | tail -1; done
