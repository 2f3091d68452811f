mkdir -p gpurun_out
export KMX_TCJ=1 KMX_TCJ_J=4 KMX_TCJ_KC=8
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/p14_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tcmulj" -c 1 \
  -o gpurun_out/p14_tcj python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/p14_ncu.log 2>&1
echo done
