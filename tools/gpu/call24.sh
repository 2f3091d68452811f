mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py -x -q > gpurun_out/t24.log 2>&1; echo pytest=$? >> gpurun_out/t24.log
