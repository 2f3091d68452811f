mkdir -p gpurun_out
KMX_FINISH_CHUNKS=1 timeout 300 python tools/paths_check.py > gpurun_out/pc18.log 2>&1; tail -1 gpurun_out/pc18.log
if grep -q "failures 0" gpurun_out/pc18.log; then
  for c in c2 c4 c1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b18_$c.json 2> gpurun_out/b18_$c.err; done
  KMX_FINISH_CHUNKS=1 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b18_c2_ch1.json 2>/dev/null
  timeout 600 python tools/sweep_c5.py --out gpurun_out/c5_18.json > gpurun_out/c5_18.log 2>&1
fi
