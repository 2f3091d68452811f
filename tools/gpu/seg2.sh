mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_kernel_paths.py -x -q -k "SEG or W1" > gpurun_out/s2_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/s2_tests.log
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/s2_c4.json 2>/dev/null; echo c4=$?
