mkdir -p gpurun_out
cd tools && timeout 600 python tcj_sweep.py --config c2 --variant 4 > ../gpurun_out/tcj_c2_v4.json 2> ../gpurun_out/tcj_c2_v4.err; cd ..
cd tools && timeout 600 python tcj_sweep.py --config c2 --variant 1 --js 1,2 --kcs 2,4,8 --nbs 2,4 > ../gpurun_out/tcj_c2_v1.json 2> ../gpurun_out/tcj_c2_v1.err; cd ..
