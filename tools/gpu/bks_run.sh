# bivariate univariate-product engine: parity + c3 timing per engine
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_batches.py tests/test_gpu_acceptance.py tests/test_gpu_bivar_mod.py -x -q -k "bivar or config3 or Bivar" > gpurun_out/b1_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/b1_tests.log
for u in 0 1 3 4 -1; do
  KMX_BKS_UNI=$u timeout 600 python bench.py --config c3 --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/b1_c3_$u.json 2>/dev/null; echo c3_$u=$?
done
