#!/usr/bin/env python
"""Parity of the CUDA path under one kernel-selection setting (environment
variables such as KMX_FINISH_WARP / KMX_TC are read once per process, so
tests/test_gpu_kernel_paths.py runs this in a subprocess per setting).

Checks, bit-exact against the oracle (oracle/ks_oracle.py, Python-int
products): every golden case generated from the reference, a BASELINE
config-2 slice (signed, n=1024), a config-4 pair (n=4096, u128), and small
and unequal shapes, for all four variants.  Exit status 0 = all equal."""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0712_4046_b200 as kmx  # noqa: E402
from oracle import ks_oracle as O  # noqa: E402
from paper_0712_4046_b200.words import ints_to_words, words_to_ints  # noqa: E402
from tests import golden_io as G  # noqa: E402


def run(v, fs, gs, b, signed=False):
    words = 1 if signed else (b + 31) // 32
    fd = torch.from_numpy(np.stack([ints_to_words(f, words, signed=signed) for f in fs]).view(np.int32)).cuda()
    gd = torch.from_numpy(np.stack([ints_to_words(g, words, signed=signed) for g in gs]).view(np.int32)).cuda()
    kb = kmx.KsBatch(v, len(fs), len(fs[0]), len(gs[0]), b, signed=signed)
    h = kb(fd, gd)
    kb.status()
    a = h.cpu().numpy().view(np.uint32)
    return [words_to_ints(a[p], signed=signed) for p in range(a.shape[0])]


def main():
    bad = 0
    for tag, f, g, b, h in G.ks_cases():
        for v in (1, 2, 3, 4):
            if run(v, [f], [g], b)[0] != h:
                print("FAIL golden", tag, v)
                bad += 1
    rng = random.Random(77)
    shapes = [(64, 1024, 1024, 32, True), (2, 4096, 4096, 128, False), (40, 16, 16, 8, False),
              (9, 300, 17, 64, False), (5, 1000, 1000, 256, False), (3, 8192, 8192, 8, False),
              (6, 700, 333, 32, True), (4, 600, 601, 30, False), (3, 2049, 2048, 20, False)]
    for B, lf, lg, b, signed in shapes:
        if signed:
            fs = [[rng.randrange(-2**31, 2**31) for _ in range(lf)] for _ in range(B)]
            gs = [[rng.randrange(-2**31, 2**31) for _ in range(lg)] for _ in range(B)]
            fs[0] = [-2**31] * lf
            gs[0] = [-2**31] * lg
            want = [O.ks_mul_signed(1, fs[p], gs[p], b, mode="native") for p in (0, B - 1)]
        else:
            fs = [[rng.randrange(1 << b) for _ in range(lf)] for _ in range(B)]
            gs = [[rng.randrange(1 << b) for _ in range(lg)] for _ in range(B)]
            fs[0] = [(1 << b) - 1] * lf
            gs[0] = [(1 << b) - 1] * lg
            want = [O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in (0, B - 1)]
        for v in (1, 2, 3, 4):
            got = run(v, fs, gs, b, signed)
            if [got[0], got[B - 1]] != want:
                print("FAIL shape", (B, lf, lg, b, signed), v)
                bad += 1
    # bivariate over Z: the reference's golden grids and a c3-shaped batch
    # (64 x 64 u16, where the univariate products take the KS path)
    Z = kmx.ring_z()
    fns = (kmx.bks_standard, kmx.bks_reciprocal, kmx.bks_negated, kmx.bks_four)
    for tag, f, g, h in G.bivar_cases():
        for v, fn in enumerate(fns, 1):
            if [list(r) for r in fn(kmx.BiPoly(tuple(map(tuple, f))), kmx.BiPoly(tuple(map(tuple, g))), Z).coeffs] != h:
                print("FAIL bivar golden", tag, v)
                bad += 1
    nrng = np.random.default_rng(33)
    F = nrng.integers(0, 1 << 16, size=(4, 64, 64), dtype=np.int64).astype(np.int32)
    Gg = nrng.integers(0, 1 << 16, size=(4, 64, 64), dtype=np.int64).astype(np.int32)
    for v in (1, 2, 3, 4):
        bb = kmx.BksBatch(v, 4, 64, 64, 16)
        hb = bb(torch.from_numpy(F).cuda(), torch.from_numpy(Gg).cuda())
        bb.status()
        if hb.cpu().tolist()[3] != O.bks(v, F[3].tolist(), Gg[3].tolist()):
            print("FAIL bivar c3 shape", v)
            bad += 1
    print("paths_check", {k: os.environ.get(k) for k in os.environ if k.startswith("KMX_")}, "failures", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
