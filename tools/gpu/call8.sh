mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cli.py -x -q > gpurun_out/t8.log 2>&1; echo pytest=$? >> gpurun_out/t8.log
for v in 4 1 3 2; do timeout 600 python tools/tc_sweep.py --config c2 --variant $v --nbs 2,3,4 > gpurun_out/tcs_c2_v$v.json 2> gpurun_out/tcs_c2_v$v.err; done
timeout 600 python tools/tc_sweep.py --config c4 --variant 4 --nbs 2,4 > gpurun_out/tcs_c4_v4.json 2> gpurun_out/tcs_c4_v4.err
timeout 600 python tools/tc_sweep.py --config c1 --variant 4 --nbs 2,4 > gpurun_out/tcs_c1_v4.json 2> gpurun_out/tcs_c1_v4.err
tail -2 gpurun_out/t8.log
