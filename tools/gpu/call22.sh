mkdir -p gpurun_out
for v in 2 4 8 16; do KMX_RECON_V=$v timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b22_c2_v$v.json 2> /dev/null; done
for v in 4 8 16; do KMX_RECON_V=$v timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/b22_c4_v$v.json 2> /dev/null; done
