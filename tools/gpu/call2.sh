set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mod.py -x -q > gpurun_out/t_mod.log 2>&1; echo mod=$? >> gpurun_out/t_mod.log
timeout 300 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python tools/sweep_c5.py --out gpurun_out/c5_sweep.json > gpurun_out/c5.log 2>&1; echo sweep=$? >> gpurun_out/c5.log
timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pack|k_tcmul|k_finish|k_recon" -c 4 -o gpurun_out/prof_c2ks4 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/ncu_f.log 2>&1; echo ncuf=$?
