# Round measurement set: full bench (CPU baseline), reference arm, ncu launch lists
# (cold + warm graph replays) and ncu --set full of the step's main kernels (warm).
mkdir -p gpurun_out/ncu
timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
bash tools/gpu/launch_list.sh
NCU_SPECS="k_fchain|chain_kernel<0, 1, 2>|2 k_bchain|chain_kernel<3, 4, 5>|2 k_l2|TcRed<.*L2Prob>|8 k_l6|TcRed<.*L6Prob>|8 k_l10|TcRed<.*L10Prob>|8 k_l7|TcRow<.*L7Prob>|8 k_msg|TcRow<.*MsgProb>|8 k_agg|agg4_kernel|8 k_seg|seg2v_kernel|10 k_a1|edge_a1_kernel|8 k_prep|edge_bwd_prep|8 k_col|colsum2_kernel|10" bash tools/gpu/ncu_graph.sh
ls gpurun_out/ncu | wc -l
