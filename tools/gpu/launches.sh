# ncu launch lists (per-kernel durations, cold, serialised) of short bench runs:
#   bash tools/gpu/launches.sh TAG "bench args" ["bench args" ...]
TAG=$1; shift
mkdir -p gpurun_out
i=0
for args in "$@"; do
  i=$((i+1))
  timeout 300 python bench.py $args --quick --steps 1 --warmup 3 > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_$i.csv \
    python bench.py $args --quick --steps 1 --warmup 3 > gpurun_out/${TAG}_$i.log 2>&1; echo "launches_$i=$? ($args)"
done
