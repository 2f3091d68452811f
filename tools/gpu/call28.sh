mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc28.log 2>&1; tail -1 gpurun_out/pc28.log
for c in c2 c4 c1; do KMX_TC_VERBOSE=1 timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b28_$c.json 2> gpurun_out/b28_$c.err; done
timeout 900 python tools/sweep_c5.py --out gpurun_out/c5_28.json > gpurun_out/c5_28.log 2>&1
