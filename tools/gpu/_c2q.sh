for p in 64 128; do KMX_TC=1 KMX_TCS=$p KMX_TCS_PERSIST=1 timeout 300 python tools/paths_check.py > gpurun_out/tcsp_paths_$p.log 2>&1; echo "persist pitch $p rc=$?"; tail -1 gpurun_out/tcsp_paths_$p.log; done
KMX_TC=1 KMX_TCS=32 KMX_TCS_PERSIST=0 timeout 300 python tools/paths_check.py > gpurun_out/tcs_paths_32.log 2>&1; echo "oneshot pitch 32 rc=$?"; tail -1 gpurun_out/tcs_paths_32.log
for pm in -1 1 0; do
KMX_TC_VERBOSE=1 KMX_TCS_PERSIST=$pm timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/tcs_c2_p$pm.json 2> gpurun_out/tcs_c2_p$pm.err; echo "PERSIST=$pm rc=$?"
grep autotune gpurun_out/tcs_c2_p$pm.err | grep "nprod=4096\|nprod=2048\|nprod=1024" | sort | uniq
python - <<PY
import json
d=json.load(open("gpurun_out/tcs_c2_p$pm.json"))
print(round(d["value"]), {k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items()}) for k,v in d["per_variant"].items()})
PY
done
