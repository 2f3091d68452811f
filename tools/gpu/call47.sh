# finish: next coefficient's prefix sums fetched early (signed coefficient output), A/B.
mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc47.log 2>&1; echo paths=$?; tail -1 gpurun_out/pc47.log
for e in "KMX_FINISH_BIAS_PREFETCH=1" "KMX_FINISH_BIAS_PREFETCH=0"; do
  env $e timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b47.json 2> /dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/b47.json'));print('$e',round(d['value']),{k:(round(v['products_per_s']),{q:round(x*1e3,1) for q,x in v['kernel_ms'].items()}) for k,v in d['per_variant'].items()})"
  cp gpurun_out/b47.json "gpurun_out/b47_$e.json"
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t47.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/t47.log
