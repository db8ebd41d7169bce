# Round measurement set: full bench (CPU baseline), reference arm, ncu launch lists
# (cold + warm graph replays), cold ncu --set full of the main kernels (DRAM traffic),
# warm ncu --set full (with source) of the dominant kernel.
mkdir -p gpurun_out/ncu
timeout 900 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
bash tools/gpu/launch_list.sh
bash tools/gpu/ncu_traffic.sh
NCU_SPECS="k_l6|TcRed<.*L6Prob>|8" bash tools/gpu/ncu_graph.sh
ls gpurun_out/ncu gpurun_out/ncu_cold | wc -l
