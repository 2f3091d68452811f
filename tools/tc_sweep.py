"""Sweep the tcgen05 multiply's tiling (KMX_TC_H, KMX_TC_KC, KMX_TC_TPC) on one
bench config and print the K2 kernel time per setting (CUDA events around the
launch, kmx_prof), plus the integer-pipe engine for reference.

usage: python tools/tc_sweep.py [--config c2] [--variant 4] [--reps 10]
"""
import argparse
import ctypes
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0712_4046_b200 as kmx  # noqa: E402
from paper_0712_4046_b200._lib import lib  # noqa: E402


def k2_ms(kb, f, g, out, reps):
    L = lib()
    prof = (ctypes.c_float * 6)()
    L.kmx_prof_enable(1)
    best = 1e30
    for _ in range(reps):
        kb(f, g, out)
        torch.cuda.synchronize()
        L.kmx_prof_read(prof, 6)
        best = min(best, prof[1])
    L.kmx_prof_enable(0)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variant", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--hs", default="1,2,3,4,6,8")
    ap.add_argument("--kcs", default="8,16,32")
    ap.add_argument("--tpcs", default="0")
    ap.add_argument("--nbs", default="2")
    ap.add_argument("--nws", default="4,8")
    ap.add_argument("--shape", default="", help="batch,n,bits (unsigned) instead of --config")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    if args.shape:
        B_, n_, b_ = map(int, args.shape.split(","))
        cfg = dict(kind="ks", batch=B_, n=n_, b=b_, signed=False)
    B, n, b, signed = cfg["batch"], cfg["n"], cfg["b"], cfg["signed"]
    words = 1 if signed else (b + 31) // 32
    rng = np.random.default_rng(1)
    f = torch.from_numpy(rng.integers(0, 2**32, size=(B, n, words), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    g = torch.from_numpy(rng.integers(0, 2**32, size=(B, n, words), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    if not signed and b % 32:
        f &= (1 << (b % 32)) - 1
        g &= (1 << (b % 32)) - 1
    kb = kmx.KsBatch(args.variant, B, n, n, b, signed=signed)
    out = kb.empty_out()
    res = []
    os.environ["KMX_TC"] = "0"
    ref = kb(f, g, out).clone()
    res.append({"engine": "imad", "k2_ms": k2_ms(kb, f, g, out, args.reps)})
    os.environ["KMX_TC"] = "1"
    for H, KC, TPC, NB, NW in itertools.product(args.hs.split(","), args.kcs.split(","), args.tpcs.split(","),
                                                args.nbs.split(","), args.nws.split(",")):
        os.environ["KMX_TC_NW"] = NW
        os.environ["KMX_TC_H"], os.environ["KMX_TC_KC"], os.environ["KMX_TC_TPC"] = H, KC, TPC
        os.environ["KMX_TC_NB"] = NB
        try:
            ms = k2_ms(kb, f, g, out, args.reps)
            ok = bool(torch.equal(out, ref))
        except Exception as e:  # unsupported tiling for this shape
            ms, ok = None, str(e)[:60]
        res.append({"H": int(H), "KC": int(KC), "TPC": int(TPC), "NB": int(NB), "NW": int(NW), "k2_ms": ms, "equal_to_imad": ok})
    for k in ("KMX_TC_H", "KMX_TC_KC", "KMX_TC_TPC", "KMX_TC_NB", "KMX_TC_NW"):
        os.environ.pop(k, None)
    os.environ["KMX_TC_VERBOSE"] = "1"
    kb(f, g, out)
    torch.cuda.synchronize()
    os.environ.pop("KMX_TC_VERBOSE")
    res.append({"engine": "tensor(default plan)", "k2_ms": k2_ms(kb, f, g, out, args.reps)})
    print(json.dumps({"config": args.shape or args.config, "variant": args.variant, "results": res}, indent=1))


if __name__ == "__main__":
    main()
