#!/usr/bin/env python
"""Reduced GPU suite for compute-sanitizer (memcheck / racecheck /
synccheck): one small call of every kernel family and every selectable
kernel path, each checked against the oracle, so the sanitizer sees the
tcgen05/mbarrier multiply, the speculative reconstruction, the warp and
chunk-parallel finishes, the bivariate and the Z/nZ paths.

  compute-sanitizer --tool racecheck python tools/sanitize_suite.py
"""
from __future__ import annotations

import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("KMX_TC_AUTOTUNE", "0")  # one launch per kernel, no timing runs


def main():
    import numpy as np
    import torch

    from oracle import ks_oracle as O
    from paper_0712_4046_b200 import BksBatch, KsBatch, ModMulBatch, _lib
    from paper_0712_4046_b200.words import ints_to_words, words_to_ints

    dev = torch.device("cuda", 0)
    rng = random.Random(11)
    checked = 0
    # (batch, n, b, signed): imad-engine shapes, tensor-core shapes, chunked finish (long streams)
    shapes = [(3, 16, 8, False), (2, 100, 64, False), (4, 256, 64, False), (2, 1024, 32, True),
              (1, 4096, 128, False)]
    for batch, n, b, signed in shapes:
        w = 1 if signed else (b + 31) // 32
        lo, hi = (-(1 << (b - 1)), 1 << (b - 1)) if signed else (0, 1 << b)
        fs = [[rng.randrange(lo, hi) for _ in range(n)] for _ in range(batch)]
        gs = [[rng.randrange(lo, hi) for _ in range(n)] for _ in range(batch)]
        fw = torch.from_numpy(np.stack([ints_to_words(f, w, signed) for f in fs]).view(np.int32)).to(dev)
        gw = torch.from_numpy(np.stack([ints_to_words(g, w, signed) for g in gs]).view(np.int32)).to(dev)
        for v in (1, 2, 3, 4):
            kb = KsBatch(v, batch, n, n, b, signed=signed, device=dev)
            h = kb(fw, gw)
            kb.status()
            hn = h.cpu().numpy().view(np.uint32)
            for p in (0, batch - 1):
                want = (O.ks_mul_signed(1, fs[p], gs[p], b, mode="native") if signed
                        else O.ks_mul(1, fs[p], gs[p], b, mode="native"))
                assert words_to_ints(hn[p], signed=signed) == want, (batch, n, b, v, p)
                checked += 1
    lx = ly = 8
    F = [[[rng.randrange(1 << 12) for _ in range(ly)] for _ in range(lx)] for _ in range(2)]
    G = [[[rng.randrange(1 << 12) for _ in range(ly)] for _ in range(lx)] for _ in range(2)]
    for v in (1, 2, 3, 4):
        bb = BksBatch(v, 2, lx, ly, 12, device=dev)
        h = bb(torch.tensor(F, dtype=torch.int32, device=dev), torch.tensor(G, dtype=torch.int32, device=dev))
        bb.status()
        assert h.cpu().tolist()[1] == O.bks(v, F[1], G[1])
        checked += 1
    n_mod = 1000003
    fm = [[rng.randrange(n_mod) for _ in range(40)] for _ in range(2)]
    gm = [[rng.randrange(n_mod) for _ in range(40)] for _ in range(2)]
    for v in (1, 2, 3, 4):
        mb = ModMulBatch(v, 2, 40, 40, n_mod, device=dev)
        h = mb(torch.tensor(fm, dtype=torch.int64, device=dev), torch.tensor(gm, dtype=torch.int64, device=dev))
        mb.status()
        assert [int(x) for x in h.cpu().numpy().view(np.uint64)[0]] == O.schoolbook_mod(fm[0], gm[0], n_mod)
        checked += 1
    torch.cuda.synchronize()
    print(f"sanitize suite ok: {checked} checks ({_lib.LIB_PATH})")


if __name__ == "__main__":
    main()
