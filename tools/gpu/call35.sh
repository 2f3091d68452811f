# Knob sweep on c2 after the lean kernels.
mkdir -p gpurun_out
for e in "KMX_FINISH_CHUNKS=1" "KMX_RECON_MINB=6" "KMX_RECON_MINB=0" "KMX_RECON_V=4" "KMX_RECON_V=16" "KMX_RECON_BIAS_SMEM=0" "KMX_RECON_SPEC=1" "KMX_PACK_PAIR=0"; do
  env $e timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b35.json 2> /dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/b35.json'));print('$e',round(d['value']),{k:(round(v['products_per_s']),{q:round(x*1e3,1) for q,x in v['kernel_ms'].items()}) for k,v in d['per_variant'].items()})"
done
