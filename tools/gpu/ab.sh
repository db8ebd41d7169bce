# A/B: default vs env toggles (quick bench, value/ms only)
mkdir -p gpurun_out
i=0
for env in ${AB_ENVS:-HMTL_X=0 HMTL_SINGLE_STREAM=1}; do
  i=$((i+1))
  echo "== $env"; env $env timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab$i.json 2> gpurun_out/ab$i.err
  python -c "import json;d=json.loads(open('gpurun_out/ab$i.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'])" || tail -25 gpurun_out/ab$i.err
done
