#!/usr/bin/env python
"""Copy one evidence run from gpurun_out/ into profiles/rNN/ (tracked).

usage: python tools/collect_evidence.py TAG [FULLTAG] [--round r02]

TAG     the tools/gpu/run.sh tag of a `tests,bench,launches` run
FULLTAG the tag of the `full` (ncu --set full, KMX_TC_AUTOTUNE=0) run; default TAG

Writes bench_default.json, bench_reference.json, launches_c2_ks4.json (summary of
the ncu launch list), ncu_full_c2_ks4.json (summary of the full capture) and
refreshes profiles/ncu_traffic.json (DRAM bytes per launch of the c2 ks4 kernels)."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = [a for a in sys.argv[1:] if not a.startswith("--")]
rnd = "r02"
if "--round" in sys.argv:
    rnd = sys.argv[sys.argv.index("--round") + 1]
    args = [a for a in args if a != rnd]
tag = args[0]
ftag = args[1] if len(args) > 1 else tag
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles", rnd)
os.makedirs(P, exist_ok=True)
shutil.copy(os.path.join(G, f"{tag}_bench.json"), os.path.join(P, "bench_default.json"))
shutil.copy(os.path.join(G, f"{tag}_reference.json"), os.path.join(P, "bench_reference.json"))
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_launches.py"), os.path.join(G, f"{tag}_launches.csv"),
                os.path.join(P, "launches_c2_ks4.json")], check=True, stdout=subprocess.DEVNULL)
full = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                       os.path.join(G, f"{ftag}_full.ncu-rep")], check=True, capture_output=True, text=True).stdout
open(os.path.join(P, "ncu_full_c2_ks4.json"), "w").write(full)
ks = json.loads(full)
role = {"k_pack": "pack_dram_bytes", "k_tc": "tcmul_dram_bytes", "k_finish": "finish_dram_bytes",
        "k_recon": "recon_dram_bytes"}
traffic = {}
for k in ks:
    for pat, name in role.items():
        if pat in k["kernel"] and name not in traffic:
            traffic[name] = k["dram_bytes"]
head = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
json.dump({"source": f"profiles/{rnd}/ncu_full_c2_ks4.json (ncu --set full, one full-batch launch each, "
                     f"bench.py --quick with KMX_TC_AUTOTUNE=0; captured on top of commit {head})",
           "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the unsplit full batch (the launch "
                   "the bench's per-kernel CUDA-event split times)",
           "configs": {"c2": {"ks4": traffic}}}, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print("collected", tag, ftag, "->", P, traffic)
