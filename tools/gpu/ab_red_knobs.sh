# A/B of the weight-gradient grid knobs (HMTL_RED_MINCH, HMTL_RED_SMS) on one GPU, two interleaved rounds
mkdir -p gpurun_out
for r in 1 2; do for kv in ${KNOBS:-"X=0" "HMTL_RED_MINCH=2" "HMTL_RED_MINCH=8" "HMTL_RED_SMS=120" "HMTL_RED_SMS=132"}; do
  env $kv timeout 300 python bench.py --no-cpu-baseline > gpurun_out/abk.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/abk.json').read().strip().splitlines()[-1]);s=d['roofline']['scopes'];print('$kv', d['value'], d['ms_per_step'], d['e2e']['value'], {k:round(v['ms_per_launch']*1000,1) for k,v in s.items() if 'grad' in k})"
done; done
