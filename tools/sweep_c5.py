#!/usr/bin/env python
"""BASELINE config 5: the crossover sweep over Z[x].

n in {16, 64, 256, 1024, 4096, 8192} x coefficient bits in {8, 32, 64, 128,
256}, unsigned uniform from seed, batch B = ceil(1e6 / (2n - 1)) pairs
(>= 1M output coefficients per point), all four KS variants.

Per point and variant: products/s (device time, CUDA-graph replay, L2
flushed between steps), the per-kernel split (CUDA events on the launch
stream), the multiply engine and its roofline fraction (live tensor / IMAD
peaks), pack/finish HBM fractions, and two parity checks: all four variants
produce bit-identical outputs on the whole batch, and pair 0 and the last pair
equal the oracle (Python-int product, oracle/ks_oracle.py ``native``).

  python tools/sweep_c5.py [--out profiles/r01_c5_sweep.json] [--steps 5]
                           [--n 16,64,...] [--bits 8,32,...] [--scale 1]

``--scale s`` multiplies every batch by s (the HBM measurement at enlarged
batch).  Writes one JSON document; prints one line per point.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

NS = (16, 64, 256, 1024, 4096, 8192)
BITS = (8, 32, 64, 128, 256)


def run_point(n, b, steps, warmup, scale, peaks, hbm, flush, dev):
    import numpy as np
    import torch

    import paper_0712_4046_b200 as kmx
    from oracle import ks_oracle as O
    from paper_0712_4046_b200 import _lib
    from paper_0712_4046_b200.words import words_to_ints

    L = _lib.lib()
    B = int(math.ceil(1e6 / (2 * n - 1))) * scale
    cfg = dict(kind="ks", batch=B, n=n, b=b, signed=False, seed=5000 + 17 * n + b,
               desc=f"c5: Z[x] u{b}, batch {B}, n={n}")
    fh, gh = bench.make_inputs(cfg)
    fd = torch.from_numpy(fh.view(np.int32)).to(dev)
    gd = torch.from_numpy(gh.view(np.int32)).to(dev)
    stream = torch.cuda.current_stream(dev)
    pt = {"n": n, "bits": b, "batch": B, "outputs": B * (2 * n - 1), "variants": {}}
    outs = {}
    prof = (ctypes.c_float * 6)()
    for v in (1, 2, 3, 4):
        op = kmx.KsBatch(v, B, n, n, b, device=dev)
        out = op.empty_out()
        for _ in range(warmup):
            op(fd, gd, out)
        op.status()
        graph, out = op.capture(fd, gd, out)
        graph.replay()
        op.status()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(steps):
            flush.fill_(1)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        op.status()
        ms = tot / steps
        kern = [0.0] * 6
        L.kmx_prof_enable(1)
        op(fd, gd, out)  # untimed: the unsplit shape's first call (plan autotuning)
        L.kmx_prof_read(prof, 6)
        for _ in range(steps):
            flush.fill_(1)
            op(fd, gd, out)
            L.kmx_prof_read(prof, 6)
            for i in range(6):
                kern[i] += prof[i]
        L.kmx_prof_enable(0)
        op.status()
        km = {nm: kern[i] / steps for i, nm in enumerate(["pack", "mul", "finish", "recon", "bias"]) if kern[i] > 0}
        if "recon" in km and "finish" not in km:  # K3 + K4 fused (k_finrec)
            km["finish+recon (fused)"] = km.pop("recon")
        prods = bench.algorithmic_products(cfg, v) * B
        eng = kmx.mul_engine(v, n, n, b)
        rec = {"products_per_s": B / (ms * 1e-3), "ms_per_step": ms, "kernel_ms": km, "mul_engine": eng,
               "limb_products_per_pair": bench.algorithmic_products(cfg, v)}
        if km.get("mul"):
            lps = prods / (km["mul"] * 1e-3)
            rec["mul_frac_of_imad_peak"] = lps / peaks["imad"]
            if eng == "tensor":
                rec["mul_frac_of_tensor_peak"] = 16.0 * lps / peaks["tensor"]
        pu = bench.pack_unpack_bytes(cfg, v)
        if "pack" in km:
            rec["pack_hbm_frac"] = pu["pack_bytes"] / (km["pack"] * 1e-3) / 1e9 / hbm
        fin_ms = km.get("finish", km.get("finish+recon (fused)"))
        rec["finish_hbm_frac"] = pu["finish_bytes"] / (fin_ms * 1e-3) / 1e9 / hbm
        pt["variants"][bench.VNAME[v]] = rec
        outs[v] = out.clone()
        del op, graph, out
    # parity: the four variants agree on the whole batch; two pairs vs the oracle
    agree = all(torch.equal(outs[1], outs[v]) for v in (2, 3, 4))
    oracle_ok = True
    for p in (0, B - 1):
        fi = bench.to_ints(fh[p:p + 1], False)[0]
        gi = bench.to_ints(gh[p:p + 1], False)[0]
        want = O.ks_mul(1, fi, gi, b, mode="native")
        got = words_to_ints(outs[4][p].cpu().numpy().view(np.uint32))
        oracle_ok = oracle_ok and got == want
    pt["variants_agree"] = bool(agree)
    pt["oracle_pairs_ok"] = bool(oracle_ok)
    base = pt["variants"]["ks1"]["products_per_s"]
    pt["speed_ratios_vs_ks1"] = {k: r["products_per_s"] / base for k, r in pt["variants"].items()}
    pt["fastest"] = max(pt["variants"], key=lambda k: pt["variants"][k]["products_per_s"])
    return pt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_c5_sweep.json"))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", default=",".join(map(str, NS)))
    ap.add_argument("--bits", default=",".join(map(str, BITS)))
    ap.add_argument("--scale", type=int, default=1)
    args = ap.parse_args()
    import torch

    import paper_0712_4046_b200 as kmx
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    peaks = {"imad": kmx.imad_peak(4096), "tensor": kmx.tc_peak(2000)}
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    mon = bench.ClockMonitor(0)
    mon.start()
    t0 = time.time()
    points = []
    for n in map(int, args.n.split(",")):
        for b in map(int, args.bits.split(",")):
            pt = run_point(n, b, args.steps, max(3, args.warmup), args.scale, peaks, hbm, flush, dev)
            points.append(pt)
            vs = pt["variants"]
            print(json.dumps({"n": n, "bits": b, "batch": pt["batch"],
                              **{k: round(r["products_per_s"], 1) for k, r in vs.items()},
                              "fastest": pt["fastest"], "agree": pt["variants_agree"],
                              "oracle": pt["oracle_pairs_ok"]}), flush=True)
    clocks = mon.stop()
    doc = {"config": "BASELINE configs[4]: crossover sweep over Z[x], unsigned uniform from seed",
           "metric": "poly products/s per KS variant (device time, CUDA-graph replay, L2 flushed)",
           "peaks": {"imad_limb_products_per_s": peaks["imad"], "tensor_u8_macs_per_s": peaks["tensor"],
                     "hbm_gbs": hbm},
           "steps": args.steps, "scale": args.scale, "clocks": clocks, "wall_s": time.time() - t0,
           "all_parity_ok": all(p["variants_agree"] and p["oracle_pairs_ok"] for p in points),
           "points": points}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps({"points": len(points), "all_parity_ok": doc["all_parity_ok"], "wall_s": doc["wall_s"]}))


if __name__ == "__main__":
    main()
