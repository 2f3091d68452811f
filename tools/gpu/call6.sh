mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t6.log 2>&1; echo pytest=$? >> gpurun_out/t6.log
for c in c2 c4 c1; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/b6_$c.json 2> gpurun_out/b6_$c.err; done
KMX_RECON_BIAS_SMEM=1 timeout 300 python bench.py --config c2 --no-cpu-baseline --no-all-variants > gpurun_out/b6_c2_bs.json 2> gpurun_out/b6_c2_bs.err
tail -2 gpurun_out/t6.log
