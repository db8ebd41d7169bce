# A/B: default library vs abuild variants (HMTL_LIB), optional env per arm
mkdir -p gpurun_out
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_$tag.json 2>/dev/null
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{t}.json"))
except Exception as e:
    print(t, "FAILED", e); sys.exit()
k = d["kernel_ms_per_step"]
top = ["k.bimg_all_kernel", "fwd.edge_msg_gemm", "fwd.edge_msg_fused", "bwd.edge_dz1_gemm", "bwd.edge_dz1_fused", "fwd.node_chain",
       "bwd.node_chain", "bwd.segsum_dst_src", "bwd.segsum_src", "fwd.agg_segsum", "bwd.force_edge_dx", "fwd.force_Qf"]
print(f"{t:10s} step {d['ms_per_step']:.4f} ms  e2e {d['e2e']['value']:.0f}", {x: k.get(x) for x in top if x in k})
PY
}
for spec in ${AB_SPECS:-"base|HMTL_X=0"}; do
  IFS='|' read -r tag envs <<< "$spec"
  run "$tag" ${envs//,/ }
done
