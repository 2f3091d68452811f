mkdir -p gpurun_out
KMX_SPLIT=1 timeout 300 python tools/paths_check.py > gpurun_out/pc19.log 2>&1; tail -1 gpurun_out/pc19.log
if grep -q "failures 0" gpurun_out/pc19.log; then
  timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b19_c2.json 2> gpurun_out/b19_c2.err
  KMX_SPLIT=0 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b19_c2_ns.json 2> /dev/null
fi
