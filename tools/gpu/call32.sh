# Recon: exact staged smem, speculative stores, register-capped instance.
mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc32.log 2>&1; echo paths=$?; tail -1 gpurun_out/pc32.log
KMX_RECON_MINB=6 timeout 300 python tools/paths_check.py > gpurun_out/pc32b.log 2>&1; echo paths6=$?; tail -1 gpurun_out/pc32b.log
for cfg in "1 5" "1 6" "1 0" "0 5" "0 0"; do set -- $cfg
  KMX_RECON_SPEC=$1 KMX_RECON_MINB=$2 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b32_s$1_m$2.json 2> /dev/null
  python -c "import json,sys;d=json.load(open('gpurun_out/b32_s$1_m$2.json'));print('s$1 m$2',round(d['value']),{k:(round(v['products_per_s']),round(v['kernel_ms'].get('recon',0)*1e3,1)) for k,v in d['per_variant'].items()})"
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t32.log 2>&1; echo pytest=$?; tail -n 2 gpurun_out/t32.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_pack_pair|k_finish_w|k_recon_par" -c 3 \
  -o gpurun_out/prof32 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/ncu32.log 2>&1; echo ncu=$?
