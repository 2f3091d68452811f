# parity subset + headline timing (one GPU call while iterating)
mkdir -p gpurun_out
TAG=${1:-q}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_batches.py tests/test_gpu_pack.py tests/test_gpu_split.py tests/test_gpu_mod.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo c2=$?
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_c2.json"))
print(round(d["value"]), {k:(round(v["products_per_s"]), {q:round(x*1e3,1) for q,x in v["kernel_ms"].items()}) for k,v in d["per_variant"].items()})
PY
