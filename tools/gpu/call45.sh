# 12-byte coefficient records as one 8-byte + one 4-byte store: parity + c1/c2 lines.
mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc45.log 2>&1; echo paths=$?; tail -1 gpurun_out/pc45.log
for c in c2 c1; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b45_$c.json 2> /dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/b45_$c.json'));print('$c',round(d['value']),{k:(round(v['products_per_s']),{q:round(x*1e3,1) for q,x in v['kernel_ms'].items()}) for k,v in d['per_variant'].items()})"
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t45.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/t45.log
