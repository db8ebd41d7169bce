# compute-sanitizer, ONE tool per call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck|initcheck
# runs a small end-to-end step sequence (eager + CUDA-graph steps of a 5-head batch) under the tool
mkdir -p gpurun_out/sanitize
TOOL=${TOOL:-memcheck}
python tools/sanitize_run.py > gpurun_out/sanitize/plain_$TOOL.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 compute-sanitizer --tool $TOOL ${SAN_ARGS} --print-limit 50 --error-exitcode 9 \
  python tools/sanitize_run.py > gpurun_out/sanitize/$TOOL.log 2>&1
echo "$TOOL rc=$?" | tee -a gpurun_out/sanitize/$TOOL.log
tail -5 gpurun_out/sanitize/$TOOL.log
