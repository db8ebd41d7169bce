# A/B of HMTL_RED_SEGX (CTA multiplier for head-segmented weight gradients) on one GPU, plus the GPU suite at segx=3
mkdir -p gpurun_out
for r in 1 2; do for x in 1 2 3 4; do
  HMTL_RED_SEGX=$x timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_${x}_${r}.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab_${x}_${r}.json').read().strip().splitlines()[-1]);s=d['roofline']['scopes'];print('segx=$x', d['value'], d['ms_per_step'], d['e2e']['value'], {k:round(v['ms_per_launch']*1000,1) for k,v in s.items() if 'wgrad' in k or 'grad' in k})"
done; done
HMTL_RED_SEGX=3 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
