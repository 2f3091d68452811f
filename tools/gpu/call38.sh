# chunk-parallel finish with the lean extraction: parity forced, c2/c1/c4 A/B.
mkdir -p gpurun_out
KMX_FINISH_CHUNKS=1 timeout 300 python tools/paths_check.py > gpurun_out/pc38.log 2>&1; echo paths_chunks=$?; tail -1 gpurun_out/pc38.log
for e in "KMX_FINISH_CHUNKS=1" "KMX_FINISH_CHUNKS=0" "KMX_NOTHING=0"; do for c in c2 c1 c4; do
  env $e timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b38.json 2> /dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/b38.json'));print('$e $c',round(d['value']),{k:(round(v['products_per_s']),{q:round(x*1e3,1) for q,x in v['kernel_ms'].items()}) for k,v in d['per_variant'].items()})"
done; done
