#!/bin/bash
# sweep multiply geometry overrides on c2 (all variants); one summary per line
for sp in 1 2 4; do for tr in 256 384 512 768; do
  KMX_SPLIT=$sp KMX_TR=$tr timeout 200 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c2 split=$sp tr=$tr', {k:(round(v['kernel_ms']['mul'],4), round(v['mul_frac_of_imad_peak'],3)) for k,v in d['per_variant'].items()})"
done; done
