mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_batches.py -x -q > gpurun_out/e4_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/e4_tests.log
for c in c2 c4; do for e in "KMX_TC_BULK=0" "KMX_TC_BULK=1"; do
  env $e timeout 600 python bench.py --config $c --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/e4.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/e4.json"))
print("$c $e", d["parity"]["oracle_ok"], round(d["value"]), {k:(round(v["products_per_s"]), round(v["kernel_ms"]["mul"]*1e3,1)) for k,v in d["per_variant"].items()})
PY
done; done
