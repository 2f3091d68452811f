#!/usr/bin/env python
"""Time the oracle port (oracle/ks_oracle.py, the CPU arm of bench.py) against
the reference package itself (kronmul, imported from /root/reference in this
container only) on the same pairs of BASELINE configs 1, 2 (unsigned part of
the bias lift) and 4, one core, and check the outputs agree.

  PYTHONDONTWRITEBYTECODE=1 python tools/port_vs_reference.py [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import bench  # noqa: E402
from kronmul import ksint  # noqa: E402
from kronmul.pack import CoeffVec  # noqa: E402
from oracle import ks_oracle as O  # noqa: E402


def main():
    rows = []
    for cname in ("c1", "c2", "c4"):
        cfg = bench.CONFIGS[cname]
        fh, gh = bench.make_inputs(cfg)
        fi = bench.to_ints(fh[:1], cfg["signed"])[0]
        gi = bench.to_ints(gh[:1], cfg["signed"])[0]
        b = cfg["b"]
        if cfg["signed"]:  # the reference takes the lifted (unsigned) inputs
            fi = [c + (1 << (b - 1)) for c in fi]
            gi = [c + (1 << (b - 1)) for c in gi]
        for v in (1, 2, 3, 4):
            fn = getattr(ksint, f"ks{v}_mul")
            F, G = CoeffVec(tuple(fi), b), CoeffVec(tuple(gi), b)
            fn(F, G)
            O.ks_mul(v, fi, gi, b, mode="karatsuba")
            t0 = time.perf_counter()
            r1 = fn(F, G)
            t1 = time.perf_counter()
            r2 = O.ks_mul(v, fi, gi, b, mode="karatsuba")
            t2 = time.perf_counter()
            assert list(r1.coeffs) == r2
            rows.append({"config": cname, "variant": f"ks{v}", "reference_s": t1 - t0, "port_s": t2 - t1,
                         "port_over_reference": (t2 - t1) / (t1 - t0)})
            print(rows[-1], flush=True)
    doc = {"what": "one pair per config and variant, one core: the oracle port's time over kronmul's own time "
                   "(outputs identical)", "rows": rows}
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02", "port_vs_reference.json")
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
