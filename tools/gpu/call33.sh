# Lean finish digit extraction; loop-free pack windows; recon speculative stores from round 2; 32-bit bias indexing.
mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc33.log 2>&1; echo paths=$?; tail -1 gpurun_out/pc33.log
for cfg in "2 1" "0 1" "2 0"; do set -- $cfg
  KMX_RECON_SPEC=$1 KMX_PACK_FAST=$2 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b33_s$1_p$2.json 2> /dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/b33_s$1_p$2.json'));print('s$1 p$2',round(d['value']),{k:(round(v['products_per_s']),{q:round(x*1e3,1) for q,x in v['kernel_ms'].items()}) for k,v in d['per_variant'].items()})"
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t33.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/t33.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_pack_pair|k_finish_w|k_recon_par" -c 3 \
  -o gpurun_out/prof33 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/ncu33.log 2>&1; echo ncu=$?
