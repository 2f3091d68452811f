mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1; echo pytest=$? >> gpurun_out/t4.log
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b4_c2.json 2> gpurun_out/b4_c2.err
KMX_RECON_WARP=1 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b4_c2_rw.json 2> gpurun_out/b4_c2_rw.err
timeout 600 python tools/sweep_c5.py --out gpurun_out/c5_4.json > gpurun_out/c5_4.log 2>&1
tail -2 gpurun_out/t4.log
