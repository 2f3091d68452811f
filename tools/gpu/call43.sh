# loop-free pack windows for every coefficient width (S >= 32): parity + c1/c2/c4 + config-5 sweep.
mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc43.log 2>&1; echo paths=$?; tail -1 gpurun_out/pc43.log
for c in c1 c2 c4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b43_$c.json 2> /dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/b43_$c.json'));print('$c',round(d['value']),{k:(round(v['products_per_s']),{q:round(x*1e3,1) for q,x in v['kernel_ms'].items()}) for k,v in d['per_variant'].items()})"
done
timeout 900 python tools/sweep_c5.py --out gpurun_out/c5_43.json > gpurun_out/c5_43.log 2>&1; echo sweep=$?; tail -1 gpurun_out/c5_43.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t43.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/t43.log
