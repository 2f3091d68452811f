mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc12.log 2>&1; echo pc=$? >> gpurun_out/pc12.log
tail -2 gpurun_out/pc12.log
if grep -q "failures 0" gpurun_out/pc12.log; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t12.log 2>&1; echo pytest=$? >> gpurun_out/t12.log
  for c in c2 c1 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b12_$c.json 2> gpurun_out/b12_$c.err; done
  tail -2 gpurun_out/t12.log
fi
