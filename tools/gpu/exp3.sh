mkdir -p gpurun_out
for e in "KMX_RECON_V=8" "KMX_RECON_V=16" "KMX_RECON_V=32" "KMX_RECON_WARP=1" "KMX_RECON_V=16 KMX_RECON_MINB=0"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/e3.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/e3.json"))
print("$e", d["parity"]["oracle_ok"], round(d["value"]), {k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items() if q in ("recon",)}) for k,v in d["per_variant"].items() if k in ("ks2","ks4")})
PY
done
for e in "KMX_RECON_V=8" "KMX_RECON_V=16" "KMX_RECON_V=32"; do
  env $e timeout 600 python bench.py --config c4 --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/e3.json 2>/dev/null
  python - <<PY
import json
d=json.load(open("gpurun_out/e3.json"))
print("c4 $e", d["parity"]["oracle_ok"], {k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items() if q in ("recon",)}) for k,v in d["per_variant"].items() if k in ("ks2","ks4")})
PY
done
