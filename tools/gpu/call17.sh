mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc17.log 2>&1; tail -1 gpurun_out/pc17.log
KMX_TCJ=1 KMX_TC=1 timeout 300 python tools/paths_check.py > gpurun_out/pc17b.log 2>&1; tail -1 gpurun_out/pc17b.log
KMX_TC_VERBOSE=1 timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/b17_c1.json 2> gpurun_out/b17_c1.err
timeout 600 python tools/sweep_c5.py --out gpurun_out/c5_17.json > gpurun_out/c5_17.log 2>&1
