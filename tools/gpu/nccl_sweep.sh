# N=4 bench under NCCL protocol / algorithm settings (tuning sweep; bench lines per setting)
mkdir -p gpurun_out
run() {
  tag=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29610 bench.py --gpus 4 > gpurun_out/sweep_$tag.json 2> gpurun_out/sweep_$tag.err
  python -c "import json;d=json.loads(open('gpurun_out/sweep_$tag.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['ms_per_step'], d.get('rank_ms_per_step'))" || tail -3 gpurun_out/sweep_$tag.err
}
run default
run ll128 NCCL_PROTO=LL128
run ll NCCL_PROTO=LL
run simple NCCL_PROTO=Simple
run ring NCCL_ALGO=Ring
run tree NCCL_ALGO=Tree
run nvls NCCL_ALGO=NVLS
run nonvls NCCL_NVLS_ENABLE=0
run ctas8 NCCL_MAX_CTAS=8
run default2
