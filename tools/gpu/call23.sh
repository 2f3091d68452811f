mkdir -p gpurun_out
timeout 300 python tools/paths_check.py > gpurun_out/pc23.log 2>&1; tail -1 gpurun_out/pc23.log
for c in c2 c4; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b23_$c.json 2> /dev/null; done
