mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_batches.py -x -q > gpurun_out/e1_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/e1_tests.log
for e in "KMX_PACK_STAGE_WORDS=12288" "KMX_PACK_STAGE_WORDS=40960"; do
  env $e timeout 600 python tools/sweep_c5.py --n 4096,8192 --bits 64,128,256 --detail --out gpurun_out/e1_c5_$e.json > /dev/null 2>&1
  python - <<PY
import json
d=json.load(open("gpurun_out/e1_c5_$e.json"))
print("$e", d["all_parity_ok"], [(p["n"],p["bits"],{k:round(v["kernel_ms"]["pack"]*1e3,1) for k,v in p["detail"].items()}) for p in d["points"]])
PY
done
for e in "KMX_RECON_SEQ=0" "KMX_RECON_SEQ=1"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/e1_c2.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/e1_c2.json"))
print("$e", d["parity"]["oracle_ok"], round(d["value"]), {k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items()}) for k,v in d["per_variant"].items()})
PY
done
