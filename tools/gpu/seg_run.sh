mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_kernel_paths.py tests/test_gpu_bench_batches.py tests/test_gpu_wide.py -x -q > gpurun_out/s1_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/s1_tests.log
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/s1_c4.json 2>/dev/null; echo c4=$?
KMX_PACK_SEG=0 timeout 600 python bench.py --config c4 --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/s1_c4_noseg.json 2>/dev/null; echo c4noseg=$?
timeout 900 python tools/sweep_c5.py --n 4096,8192 --out gpurun_out/s1_c5.json > gpurun_out/s1_c5.log 2>&1; echo c5=$?; tail -1 gpurun_out/s1_c5.log
