# A/B the step with engine ablation bits (timing experiments; wrong numbers by design)
mkdir -p gpurun_out
for dbg in 0 4 2 6 1; do
  HMTL_TC_DEBUG=$dbg timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/ab_dbg$dbg.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_dbg$dbg.json')); k=d['kernel_ms_per_step']
print('dbg=$dbg', d['ms_per_step'], {x: k.get(x) for x in ('fwd.edge_msg_fused','bwd.edge_dz1_fused','bwd.segsum_src','fwd.agg_fix')})"
done
