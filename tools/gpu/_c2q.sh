for ks in 128 40 27 20; do
KMX_TCS_KS=$ks timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/tcs_c2_ks$ks.json 2> gpurun_out/tcs_c2_ks$ks.err; echo "KS=$ks rc=$?"
python - <<PY
import json
d=json.load(open("gpurun_out/tcs_c2_ks$ks.json"))
print(round(d["value"]), {k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items()}) for k,v in d["per_variant"].items()})
PY
done
