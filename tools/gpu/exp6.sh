mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_bench_batches.py -x -q 2>&1 | tail -1
for c in c2 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-per-config --no-c5 > gpurun_out/e6.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e6.json')); print('$c', d['parity']['oracle_ok'], round(d['value']), {k:(round(v['products_per_s']), round(v['kernel_ms']['mul']*1e3,1), v['roofline']['mul_plan'].get('TPC')) for k,v in d['per_variant'].items()})"
done
timeout 900 python tools/sweep_c5.py --n 4096,8192 --out gpurun_out/e6_c5.json > gpurun_out/e6_c5.log 2>&1; tail -11 gpurun_out/e6_c5.log
