# per-kernel durations of graph steps: cold (ncu default cache flush) and warm (--cache-control none)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 4 --graph > gpurun_out/ncu_launch.log 2>&1; echo "cold rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 1000 --csv \
  --log-file gpurun_out/launches_warm.csv python tools/profile_step.py --steps 4 --graph > gpurun_out/ncu_launch_warm.log 2>&1; echo "warm rc=$?"
