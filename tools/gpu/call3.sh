mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t3.log 2>&1; echo pytest=$? >> gpurun_out/t3.log
for c in c2 c1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b3_$c.json 2> gpurun_out/b3_$c.err; done
timeout 600 python tools/sweep_c5.py --n 16,64,256,1024 --out gpurun_out/c5_small3.json > gpurun_out/c5s3.log 2>&1
KMX_TC=0 timeout 600 python tools/sweep_c5.py --n 16,64,256 --out gpurun_out/c5_small3_imad.json > gpurun_out/c5s3i.log 2>&1
tail -2 gpurun_out/t3.log
