mkdir -p gpurun_out
KMX_TC_VERBOSE=1 timeout 300 python tools/paths_check.py > gpurun_out/pc9.log 2> gpurun_out/pc9.err; echo pc=$? >> gpurun_out/pc9.log
tail -3 gpurun_out/pc9.log; grep -c kmx_tcj gpurun_out/pc9.err
if grep -q "failures 0" gpurun_out/pc9.log; then
  KMX_TC_VERBOSE=1 timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b9_c2.json 2> gpurun_out/b9_c2.err
  timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/b9_c1.json 2> gpurun_out/b9_c1.err
  timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/b9_c4.json 2> gpurun_out/b9_c4.err
  for J in 2 4 8; do KMX_TCJ_J=$J timeout 300 python bench.py --config c2 --no-cpu-baseline --no-all-variants > gpurun_out/b9_c2_J$J.json 2>/dev/null; done
fi
