for env in "HMTL_X=0" "HMTL_NO_A1=1" "HMTL_X=0" "HMTL_NO_A1=1" "HMTL_X=0" "HMTL_NO_A1=1" "HMTL_SINGLE_STREAM=1" "HMTL_SINGLE_STREAM=1 HMTL_NO_A1=1"; do
  echo "== $env: $(env $env timeout 120 python tools/repro_bench_warmup.py 30 2>&1 | tail -1)"
done
