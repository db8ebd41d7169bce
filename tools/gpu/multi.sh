# multi-GPU: NCCL equivalence test + bench at N = 2..$NG
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_dist.py -x -q 2>&1 | tail -3
for n in 1 2 4 8; do
  [ $n -gt $NG ] && break
  if [ $n -eq 1 ]; then timeout 600 python bench.py --no-cpu-baseline > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err
  else HMTL_COMM_LOG=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus $n > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err; fi
  python -c "import json;d=json.loads(open('gpurun_out/scale_$n.json').read().strip().splitlines()[-1]);print($n, d['value'], d['ms_per_step'], d['e2e']['value'], d.get('rank_ms_per_step'), d['config']['per_gpu_batch'], d.get('comm'))" || tail -5 gpurun_out/scale_$n.err
done
