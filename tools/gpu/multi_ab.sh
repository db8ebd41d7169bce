# N-GPU bench under env variants: value, ms, per-rank ms
NG=${NG:-4}
i=0
for env in ${AB_ENVS:-HMTL_X=0}; do
  i=$((i+1))
  env $env timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $((29700+i)) bench.py --gpus $NG --no-cpu-baseline > gpurun_out/mab$i.json 2> gpurun_out/mab$i.err
  echo "$env: $(python -c "import json;d=json.loads(open('gpurun_out/mab$i.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d.get('rank_ms_per_step'))" 2>&1 | tail -1)"
done
