# e2e with / without the between-step L2 flush (same box)
mkdir -p gpurun_out
for env in HMTL_X=0 HMTL_E2E_NOFLUSH=1; do
  env $env timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/e2e_$env.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/e2e_$env.json').read().strip().splitlines()[-1]);print('$env', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
