#!/usr/bin/env python
"""Derive GPU AUTO bands (modpoly.AutoThresholds) from the config-5 sweep.

The reference's AUTO (modpoly.py:79-92) is a length-only band lookup: ks1 up
to ks1_max_length, ks3 up to ks3_max_length, ks4 beyond.  This reads
profiles/r01/c5_sweep_final6.json and, over coefficient widths up to --max-bits
(word-sized moduli: the (Z/nZ)[x] front end has b <= 64), picks the band
edges that minimise the total time lost against the per-point fastest
variant, searching edges over the swept lengths.

  python tools/calibrate_auto.py [--sweep profiles/r01/c5_sweep_final6.json] [--max-bits 64]
"""
import argparse
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", default=os.path.join(ROOT, "profiles", "r01_c5_sweep.json"))
    ap.add_argument("--max-bits", type=int, default=64)
    args = ap.parse_args()
    doc = json.load(open(args.sweep))
    pts = [p for p in doc["points"] if p["bits"] <= args.max_bits]
    lengths = sorted({p["n"] for p in pts})
    edges = [0] + lengths

    def lost(e1, e3):
        tot = 0.0
        for p in pts:
            v = "ks1" if p["n"] <= e1 else ("ks3" if p["n"] <= e3 else "ks4")
            t = {k: 1.0 / r["products_per_s"] for k, r in p["variants"].items()}
            tot += t[v] / min(t.values()) - 1.0
        return tot

    best = min(((lost(a, b), a, b) for a in edges for b in edges if b >= a), key=lambda x: x[0])
    print(json.dumps({"ks1_max_length": best[1], "ks3_max_length": best[2],
                      "mean_slowdown_vs_best": best[0] / len(pts),
                      "fastest_per_point": {f"n{p['n']}_b{p['bits']}": p["fastest"] for p in pts}}, indent=1))


if __name__ == "__main__":
    main()
