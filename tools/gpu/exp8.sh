timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_batches.py -x -q -k "host or bench_config" 2>&1 | tail -1
for e in "KMX_HOST_PIPE=0" "KMX_HOST_CHUNK_MB=4" "KMX_HOST_CHUNK_MB=2" "KMX_HOST_CHUNK_MB=3" "KMX_HOST_CHUNK_MB=6"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 --no-all-variants > gpurun_out/e8.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e8.json')); print('$e', round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3), d['e2e']['equals_device_output'])"
done
