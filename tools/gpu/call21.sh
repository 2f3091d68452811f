mkdir -p gpurun_out
for c in c1 c4; do KMX_SPLIT=1 timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b21_${c}_s1.json 2> /dev/null; timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b21_${c}_s0.json 2> /dev/null; done
