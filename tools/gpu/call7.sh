mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bivar_mod.py tests/test_gpu_mod.py -x -q > gpurun_out/t7a.log 2>&1; echo pytest=$? >> gpurun_out/t7a.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t7.log 2>&1; echo pytest=$? >> gpurun_out/t7.log
tail -2 gpurun_out/t7a.log gpurun_out/t7.log
