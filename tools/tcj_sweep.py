"""Sweep the chunked tensor-core multiply (kmx_tcj.cu) settings on one bench
config: K2 time per (J, H0, KC, NB, NW) next to the tiled kernel (KMX_TCJ=0),
each checked bit-equal to the integer pipe.
usage: python tools/tcj_sweep.py [--config c2] [--variant 4]"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tc_sweep import k2_ms  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0712_4046_b200 as kmx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variant", type=int, default=4)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--js", default="2,4")
    ap.add_argument("--hs", default="0")
    ap.add_argument("--kcs", default="4,8,16")
    ap.add_argument("--nbs", default="2,3,4")
    ap.add_argument("--nws", default="4,8")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
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
    os.environ["KMX_TC"] = "0"
    ref = kb(f, g, out).clone()
    os.environ["KMX_TC"] = "1"
    res = []
    os.environ["KMX_TCJ"] = "0"
    res.append({"kernel": "tiled k_tcmul", "k2_ms": k2_ms(kb, f, g, out, args.reps)})
    os.environ["KMX_TCJ"] = "1"
    for J, H, KC, NB, NW in itertools.product(args.js.split(","), args.hs.split(","), args.kcs.split(","),
                                              args.nbs.split(","), args.nws.split(",")):
        os.environ.update({"KMX_TCJ_J": J, "KMX_TCJ_H": H, "KMX_TCJ_KC": KC, "KMX_TCJ_NB": NB, "KMX_TCJ_NW": NW})
        try:
            ms = k2_ms(kb, f, g, out, args.reps)
            ok = bool(torch.equal(out, ref))
        except Exception as e:
            ms, ok = None, str(e)[:60]
        res.append({"J": int(J), "H0": int(H), "KC": int(KC), "NB": int(NB), "NW": int(NW), "k2_ms": ms, "equal": ok})
    print(json.dumps({"config": args.config, "variant": args.variant, "results": res}, indent=1))


if __name__ == "__main__":
    main()
