mkdir -p gpurun_out
KMX_SPLIT=1 KMX_SPLIT_WAYS=3 timeout 300 python tools/paths_check.py > gpurun_out/pc20.log 2>&1; tail -1 gpurun_out/pc20.log
if grep -q "failures 0" gpurun_out/pc20.log; then
  for w in 2 3 4; do KMX_SPLIT_WAYS=$w timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b20_c2_w$w.json 2> /dev/null; done
  KMX_SPLIT_WAYS=2 timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/b20_c3.json 2> /dev/null
fi
