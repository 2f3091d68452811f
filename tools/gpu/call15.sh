mkdir -p gpurun_out
KMX_TCJ=1 KMX_TC=1 timeout 300 python tools/paths_check.py > gpurun_out/pc15.log 2>&1; tail -1 gpurun_out/pc15.log
cd tools && timeout 600 python tcj_sweep.py --config c2 --variant 4 --js 2,4,8 --kcs 4,8 --nbs 2,3 --nws 4,8 > ../gpurun_out/tcj15_c2_v4.json 2>&1; cd ..
cd tools && timeout 600 python tcj_sweep.py --config c2 --variant 1 --js 1,2 --kcs 2,4 --nbs 2 --nws 4,8 > ../gpurun_out/tcj15_c2_v1.json 2>&1; cd ..
cd tools && timeout 600 python tcj_sweep.py --config c1 --variant 4 --js 2,4 --kcs 4,8 --nbs 2 --nws 4,8 > ../gpurun_out/tcj15_c1_v4.json 2>&1; cd ..
