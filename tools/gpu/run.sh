#!/usr/bin/env bash
# One entry point for the GPU-box jobs of this repo (run it through gpurun):
#
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/gpu/run.sh MODE [TAG]'
#
# MODE (several may be given, comma-separated; outputs land in gpurun_out/):
#   tests     pytest -m gpu plus smoke()                      -> TAG_tests.log, TAG_smoke.log
#   bench     default bench line (all configs) + reference arm -> TAG_bench.json, TAG_reference.json
#   sweep     config-5 crossover sweep, every point checked   -> TAG_c5.json
#   launches  ncu launch list of the default command           -> TAG_launches.csv
#   full      ncu --set full of the c2 ks4 hot kernels         -> TAG_full.ncu-rep
#   sanitize  compute-sanitizer memcheck/racecheck/synccheck   -> TAG_san_*.log
#             over tools/sanitize_suite.py (reduced suite); NOTE: the round-2
#             GPU pool refuses compute-sanitizer (exit 86, "closed on this
#             pool"), so this mode only runs where the tool is allowed
# After a `tests,bench,launches` run (TAG) and a `KMX_TC_AUTOTUNE=0 ... full` run (FULLTAG),
# `python tools/collect_evidence.py TAG FULLTAG` copies the tracked evidence set into profiles/rNN/.
# Each step runs only after the previous one of the same mode exited 0
# (profilers never run on a command that has not already passed without them).
set -u
MODES=${1:-tests,bench}
TAG=${2:-run}
O=gpurun_out
mkdir -p $O
has() { case ",$MODES," in *",$1,"*) return 0;; *) return 1;; esac; }
if has tests; then
  timeout 2400 python -m pytest tests -m gpu -x -q > $O/${TAG}_tests.log 2>&1; echo "pytest=$?" | tee -a $O/${TAG}_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke=$?" | tee -a $O/${TAG}_smoke.log
  tail -n 3 $O/${TAG}_tests.log
fi
if has bench; then
  timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench=$?"
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_reference.json 2> $O/${TAG}_reference.err; echo "reference=$?"
fi
if has sweep; then
  timeout 1500 python tools/sweep_c5.py --out $O/${TAG}_c5.json > $O/${TAG}_c5.log 2>&1; echo "sweep=$?"
fi
if has launches; then
  timeout 300 python bench.py --steps 3 --warmup 3 --quick > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --quick > $O/${TAG}_launches.log 2>&1; echo "launches=$?"
fi
if has full; then
  KREGEX=${KREGEX:-"regex:k_pack|k_tcmul|k_tcswz|k_finish|k_recon|k_kara"}
  timeout 300 python bench.py --steps 3 --warmup 3 --quick > /dev/null 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k "$KREGEX" -c ${NCU_COUNT:-6} \
    -o $O/${TAG}_full python bench.py --steps 3 --warmup 3 --quick > $O/${TAG}_full.log 2>&1; echo "full=$?"
fi
if has sanitize; then
  for tool in memcheck racecheck synccheck; do
    timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_suite.py \
      > $O/${TAG}_san_$tool.log 2>&1; echo "sanitize_$tool=$?" | tee -a $O/${TAG}_san_$tool.log
  done
fi
echo done
