mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc30.log 2>&1; tail -1 gpurun_out/pc30.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t30.log 2>&1; echo pytest=$? >> gpurun_out/t30.log; tail -n 2 gpurun_out/t30.log
for c in c2 c1 c4; do KMX_TC_VERBOSE=1 timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b30_$c.json 2> gpurun_out/b30_$c.err; done
timeout 900 python tools/sweep_c5.py --out gpurun_out/c5_30.json > gpurun_out/c5_30.log 2>&1
