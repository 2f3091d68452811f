mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t5.log 2>&1; echo pytest=$? >> gpurun_out/t5.log
for c in c2 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b5_$c.json 2> gpurun_out/b5_$c.err; done
KMX_TC_VERBOSE=1 timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 3 --no-all-variants --variant 2 > gpurun_out/b5_c4v.json 2> gpurun_out/b5_c4v.err
timeout 600 python tools/sweep_c5.py --n 1024,4096,8192 --out gpurun_out/c5_5.json > gpurun_out/c5_5.log 2>&1
tail -2 gpurun_out/t5.log
