mkdir -p gpurun_out
for sh in "32,4096,128:4" "123,4096,64:4" "62,8192,32:4" "123,4096,32:4" "489,1024,128:4" "123,4096,64:2"; do
  shape=${sh%%:*}; v=${sh##*:}
  KMX_TC_VERBOSE=1 timeout 600 python tools/tc_sweep.py --shape $shape --variant $v --hs 3 --kcs 16 --nbs 2 --nws 4 --reps 3 > gpurun_out/tcs27_${shape//,/_}_v$v.json 2> gpurun_out/tcs27_${shape//,/_}_v$v.err
done
for c in c2 c4 c1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b27_$c.json 2> /dev/null; done
timeout 600 python tools/sweep_c5.py --out gpurun_out/c5_27.json > gpurun_out/c5_27.log 2>&1
