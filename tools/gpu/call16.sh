mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc16.log 2>&1; tail -1 gpurun_out/pc16.log
for c in c1 c2; do KMX_TC_VERBOSE=1 timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b16_$c.json 2> gpurun_out/b16_$c.err; done
timeout 600 python tools/sweep_c5.py --out gpurun_out/c5_16.json > gpurun_out/c5_16.log 2>&1
