mkdir -p gpurun_out
for sh in "32,4096,128:4" "123,4096,64:4" "62,8192,32:4" "123,4096,32:4" "489,1024,128:4" "32,4096,128:3" "123,4096,64:2"; do
  shape=${sh%%:*}; v=${sh##*:}
  KMX_TC_VERBOSE=1 timeout 600 python tools/tc_sweep.py --shape $shape --variant $v --hs 2,3,4,6,8 --kcs 8,16 --nbs 2 --nws 4,8 --reps 3 > gpurun_out/tcs26_${shape//,/_}_v$v.json 2> gpurun_out/tcs26_${shape//,/_}_v$v.err
done
