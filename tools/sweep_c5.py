#!/usr/bin/env python
"""BASELINE config 5: the crossover sweep over Z[x] (standalone form of the
``c5`` block bench.py prints in its default line).

n in {16, 64, 256, 1024, 4096, 8192} x coefficient bits in {8, 32, 64, 128,
256}, unsigned uniform from seed, batch B = ceil(1e6 / (2n - 1)) pairs
(>= 1M output coefficients per point) times ``--scale``.
Per point and variant: products/s (device time, CUDA-graph replay, L2
flushed), the kernel split, K2's roofline and the pack / finish /
reconstruction HBM fractions (``--detail``), and the parity flag: the four
variants bit-identical on the whole batch and the oracle on the first and
last pair.

  python tools/sweep_c5.py [--out FILE] [--steps 5] [--n 16,64] [--bits 8,32] [--scale 1] [--detail]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c5_sweep.json"))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", default=",".join(map(str, bench.C5_NS)))
    ap.add_argument("--bits", default=",".join(map(str, bench.C5_BITS)))
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--detail", action="store_true")
    args = ap.parse_args()
    g = bench.Gpu(0)
    mon = bench.ClockMonitor(0)
    mon.start()
    doc = bench.c5_summary(g, args.steps, max(3, args.warmup), args.scale,
                           tuple(map(int, args.n.split(","))), tuple(map(int, args.bits.split(","))),
                           detail=args.detail)
    doc["clocks"] = mon.stop()
    doc["peaks"] = {"imad_limb_products_per_s": g.imad, "tensor_u8_macs_per_s": g.tensor, "hbm_gbs": g.hbm}
    for p in doc["points"]:
        print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in p.items()
                          if k not in ("detail", "mul_frac", "hbm_frac", "mul_engine")}), flush=True)
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps({"points": len(doc["points"]), "all_parity_ok": doc["all_parity_ok"], "wall_s": doc["wall_s"]}))


if __name__ == "__main__":
    main()
