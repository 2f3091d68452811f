mkdir -p gpurun_out
for e in "KMX_FUSE=0" "KMX_FUSE=1" "KMX_SPLIT=0" "KMX_SPLIT_WAYS=4 KMX_SPLIT=1"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/e2.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/e2.json"))
print("$e", d["parity"]["oracle_ok"], round(d["value"]), {k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items()}) for k,v in d["per_variant"].items()})
PY
done
