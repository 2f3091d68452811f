mkdir -p gpurun_out
KMX_SPLIT_STAGGER=1 timeout 300 python tools/paths_check.py > gpurun_out/pc29.log 2>&1; tail -1 gpurun_out/pc29.log
for w in 2 3 4; do KMX_SPLIT_STAGGER=1 KMX_SPLIT_WAYS=$w timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b29_w$w.json 2> /dev/null; done
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/b29_ns.json 2> /dev/null
