# Round-end evidence: tests, smoke, bench lines (default + reference arm + c1/c3/c4),
# the config-5 sweep, an ncu launch list of the default command and one
# ncu --set full capture of the hot kernels.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f6_tests.log 2>&1; echo pytest=$? >> gpurun_out/f6_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1; echo smoke=$? >> gpurun_out/f6_smoke.log
timeout 600 python bench.py > gpurun_out/f6_bench_default.json 2> gpurun_out/f6_bench_default.err; echo bench=$? >> gpurun_out/f6_bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f6_bench_reference.json 2> gpurun_out/f6_bench_reference.err
for c in c1 c3 c4; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/f6_bench_$c.json 2> gpurun_out/f6_bench_$c.err; done
timeout 900 python tools/sweep_c5.py --out gpurun_out/f6_c5_sweep.json > gpurun_out/f6_c5.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/f6_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f6_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/f6_ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pack|k_tcmul|k_finish|k_recon" -c 4 \
  -o gpurun_out/f6_prof python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/f6_ncu_f.log 2>&1
echo done
tail -n 2 gpurun_out/f6_tests.log; tail -n 2 gpurun_out/f6_smoke.log
