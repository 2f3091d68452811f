for e in "KMX_HOST_CHUNK_MB=4" "KMX_HOST_CHUNK_MB=2" "KMX_HOST_CHUNK_MB=1" "KMX_HOST_CHUNK_MB=8"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --no-per-config --no-c5 --no-all-variants > gpurun_out/e7.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e7.json')); print('$e', round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3), d['e2e']['equals_device_output'])"
done
