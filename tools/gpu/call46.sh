# ncu --set full of the final finish and reconstruction kernels (c2 ks4).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_finish_w|k_recon_par" -c 2 \
  -o gpurun_out/prof46 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-all-variants > gpurun_out/ncu46.log 2>&1; echo ncu=$?
