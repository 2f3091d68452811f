# Re-entry check of HEAD on a fresh box: gpu tests, smoke, default bench.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t31.log 2>&1; echo pytest=$? >> gpurun_out/t31.log; tail -n 3 gpurun_out/t31.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s31.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/b31_default.json 2> gpurun_out/b31_default.err; echo bench=$?
