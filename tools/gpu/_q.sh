for cf in 0 -1; do KMX_PACK_CF=$cf timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/cf_c4_$cf.json 2> gpurun_out/cf_c4_$cf.err; echo "c4 cf=$cf rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/cf_c4_$cf.json"))
print({k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items()}) for k,v in d["per_variant"].items()}, d.get("parity"))
PY
done
