mkdir -p gpurun_out
KMX_KARA_MIN=600 timeout 600 python tools/paths_check.py > gpurun_out/k1_paths600.log 2>&1; echo paths600=$?; tail -3 gpurun_out/k1_paths600.log
KMX_KARA_MIN=300 KMX_TC=0 timeout 600 python tools/paths_check.py > gpurun_out/k1_paths300.log 2>&1; echo paths300=$?; tail -3 gpurun_out/k1_paths300.log
timeout 900 python -m pytest tests/test_gpu_bench_batches.py -x -q > gpurun_out/k1_bb.log 2>&1; echo bb=$?; tail -3 gpurun_out/k1_bb.log
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/k1_c4.json 2>gpurun_out/k1_c4.err; echo c4=$?
for km in 8000 16000 30000; do KMX_KARA_MIN=$km timeout 600 python bench.py --config c4 --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/k1_c4_$km.json 2>/dev/null; echo c4_$km=$?; done
timeout 900 python tools/sweep_c5.py --n 4096,8192 --out gpurun_out/k1_c5.json > gpurun_out/k1_c5.log 2>&1; echo c5=$?; tail -12 gpurun_out/k1_c5.log
