mkdir -p gpurun_out
KMX_RECON_BIAS_SMEM=0 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b13_c2_bs0.json 2>/dev/null
KMX_FINREC=0 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b13_c2_nofuse.json 2>/dev/null
timeout 600 python tools/sweep_c5.py --n 16,64,256,1024 --out gpurun_out/c5_13.json > gpurun_out/c5_13.log 2>&1
KMX_FINREC=0 timeout 600 python tools/sweep_c5.py --n 16,64,256,1024 --out gpurun_out/c5_13_nofuse.json > gpurun_out/c5_13n.log 2>&1
