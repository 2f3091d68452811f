"""Generate golden input/output vectors from the REFERENCE package itself.

Run in the builder container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``kronmul`` from /root/reference/pkg/src (read-only; bytecode
writing disabled) and records, for seeded inputs, the exact outputs of
``ks1_mul .. ks4_mul`` (pkg/src/kronmul/ksint.py:219-348), the pack
functions (pack.py:79-110), ``reconstruct_overlapped`` (ksint.py:182-195) and
``bks_*`` with ``ring_z()`` (bipoly.py:177-278).  The fixtures are committed;
the GPU box never reads /root/reference.
"""
import gzip
import json
import os
import random
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import kronmul as K  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
VARIANTS = {1: K.ks1_mul, 2: K.ks2_mul, 3: K.ks3_mul, 4: K.ks4_mul}
BVARIANTS = {1: K.bks_standard, 2: K.bks_reciprocal, 3: K.bks_negated, 4: K.bks_four}


def hexs(vals):
    return [format(int(v), "x") for v in vals]


def ks_case(f, g, b, tag):
    F, G = K.CoeffVec(tuple(f), b), K.CoeffVec(tuple(g), b)
    outs = {v: fn(F, G).coeffs for v, fn in VARIANTS.items()}
    # the four reference variants agree bit for bit; store the product once
    assert len({outs[v] for v in outs}) == 1, tag
    return {"tag": tag, "b": b, "f": hexs(f), "g": hexs(g), "h": hexs(outs[1])}


def main():
    rng = random.Random(20260101)
    cases = []
    # reference worked example (tests/test_ksint.py:12-14)
    cases.append(ks_case([274, 610, 887, 621], [553, 298, 424, 790], 10, "worked_example"))
    # zero vector and single coefficient (tests/test_ksint.py:64-69)
    cases.append(ks_case([0, 0, 0], [7, 21, 30], 5, "zeros"))
    cases.append(ks_case([9], [13], 4, "single"))
    # all-max inputs (overlapped +1-bit law regime, tests/test_pack.py:129-137)
    for b in (1, 4, 17, 31, 32, 33, 48, 64, 65, 128):
        for L in (1, 2, 3, 5, 8, 100):
            top = (1 << b) - 1
            cases.append(ks_case([top] * L, [top] * L, b, f"allmax_b{b}_L{L}"))
    # random, including unequal lengths (tests/test_acceptance.py:57-74)
    for i in range(160):
        b = rng.choice([1, 2, 3, 7, 8, 9, 15, 16, 17, 24, 31, 32, 33, 40, 48, 63, 64, 65,
                        96, 100, 127, 128, 129, 200, 256])
        lf = max(1, int(300 ** rng.random()))
        lg = lf if i % 3 == 0 else max(1, int(300 ** rng.random()))
        f = [rng.randrange(1 << b) for _ in range(lf)]
        g = [rng.randrange(1 << b) for _ in range(lg)]
        cases.append(ks_case(f, g, b, f"random_{i}"))
    # exhaustive tiny lengths 1..3 with coefficients < 8 (sampled)
    tiny = []
    for L in (1, 2, 3):
        for _ in range(40):
            tiny.append([rng.randrange(8) for _ in range(L)])
    for i in range(120):
        f, g = rng.choice(tiny), rng.choice(tiny)
        cases.append(ks_case(f, g, 3, f"tiny_{i}"))
    # BASELINE config-1 shape (n=256, b=64), 4 pairs; config-4 shape (n=4096, b=128) 1 pair
    for i in range(4):
        f = [rng.randrange(1 << 64) for _ in range(256)]
        g = [rng.randrange(1 << 64) for _ in range(256)]
        cases.append(ks_case(f, g, 64, f"c1_pair{i}"))
    f = [rng.randrange(1 << 128) for _ in range(4096)]
    g = [rng.randrange(1 << 128) for _ in range(4096)]
    cases.append(ks_case(f, g, 128, "c4_pair0"))

    with gzip.open(os.path.join(HERE, "ks_golden.json.gz"), "wt") as fh:
        json.dump(cases, fh)

    # pack KATs and randomized packs (tests/test_pack.py)
    packs = []
    for coeffs, b, w in [((1, 2, 3), 8, 8), ((3, 2, 1), 4, 4), ((9,), 4, 6), ((11,), 4, 4),
                         ((135, 200, 77), 8, 5), ((274, 610, 887, 621), 10, 12)]:
        v = K.CoeffVec(coeffs, b)
        packs.append({"c": hexs(coeffs), "b": b, "w": w,
                      "pack": int(K.pack(v, w)), "rev": int(K.pack_reversed(v, w)),
                      "neg": K.pack_negated(v, w).value, "nrev": K.pack_negated_reversed(v, w).value})
    for _ in range(200):
        b = rng.randrange(1, 70)
        L = rng.randrange(1, 20)
        coeffs = tuple(rng.randrange(1 << b) for _ in range(L))
        w = rng.randrange((b + 1) // 2, 2 * b + 10)
        v = K.CoeffVec(coeffs, b)
        packs.append({"c": hexs(coeffs), "b": b, "w": w,
                      "pack": int(K.pack(v, w)), "rev": int(K.pack_reversed(v, w)),
                      "neg": K.pack_negated(v, w).value, "nrev": K.pack_negated_reversed(v, w).value})
    for p in packs:
        for key in ("pack", "rev", "neg", "nrev"):
            p[key] = str(p[key])
    with gzip.open(os.path.join(HERE, "pack_golden.json.gz"), "wt") as fh:
        json.dump(packs, fh)

    # reconstruction KATs (tests/test_ksint.py:115-127) + random round trips
    recs = [{"fwd": [5, 2], "rev": [2, 5], "w": 3, "h": [21]},
            {"fwd": [3, 3, 7, 0], "rev": [0, 4, 3, 6], "w": 3, "h": [3, 11, 6]}]
    for _ in range(300):
        w = rng.randrange(2, 140)
        count = rng.randrange(1, 60)
        top = (1 << w) * ((1 << w) - 1)
        vals = [rng.randrange(top) for _ in range(count)]
        fv = sum(h << (i * w) for i, h in enumerate(vals))
        rv = sum(h << ((count - 1 - i) * w) for i, h in enumerate(vals))
        m = (1 << w) - 1
        fwd = [(fv >> (i * w)) & m for i in range(count + 1)]
        rev = [(rv >> (i * w)) & m for i in range(count + 1)][::-1]
        got = K.reconstruct_overlapped(K.OverlapDigits(tuple(fwd), tuple(rev), w))
        recs.append({"fwd": hexs(fwd), "rev": hexs(rev), "w": w, "h": hexs(got.coeffs)})
    recs[0] = {k: (hexs(v) if isinstance(v, list) else v) for k, v in recs[0].items()}
    recs[1] = {k: (hexs(v) if isinstance(v, list) else v) for k, v in recs[1].items()}
    with gzip.open(os.path.join(HERE, "recon_golden.json.gz"), "wt") as fh:
        json.dump(recs, fh)

    # bivariate over Z (tests/test_bipoly.py): example + random signed grids +
    # one BASELINE config-3 sized pair.  A fast exact UniMul is plugged in
    # through the reference's own callback (bipoly.py:23, :121-125); the
    # bks_* reductions themselves are the reference code.
    Z = K.ring_z()

    def fastmul(a, b):
        r = np.convolve(np.asarray(a, dtype=object), np.asarray(b, dtype=object))
        return [int(x) for x in r]

    bcases = []

    def bcase(f, g, tag, mul=None):
        F = K.BiPoly(tuple(map(tuple, f)))
        G = K.BiPoly(tuple(map(tuple, g)))
        outs = {v: fn(F, G, Z, mul).coeffs for v, fn in BVARIANTS.items()}
        assert len({outs[v] for v in outs}) == 1, tag
        return {"tag": tag, "f": f, "g": g, "h": [list(r) for r in outs[1]]}

    bcases.append(bcase([[1, 3], [2, 4]], [[5, 0], [6, 1]], "example"))
    bcases.append(bcase([[3]], [[5]], "single"))
    bcases.append(bcase([[2], [3], [4]], [[1], [5], [9]], "const_in_y"))
    for i in range(60):
        lx, ly = rng.randrange(1, 12), rng.randrange(1, 12)
        f = [[rng.randrange(-99, 100) for _ in range(ly)] for _ in range(lx)]
        g = [[rng.randrange(-99, 100) for _ in range(ly)] for _ in range(lx)]
        bcases.append(bcase(f, g, f"random_{i}"))
    for i in range(2):
        f = [[rng.randrange(1 << 16) for _ in range(64)] for _ in range(64)]
        g = [[rng.randrange(1 << 16) for _ in range(64)] for _ in range(64)]
        bcases.append(bcase(f, g, f"c3_pair{i}", fastmul))
    with gzip.open(os.path.join(HERE, "bivar_golden.json.gz"), "wt") as fh:
        json.dump(bcases, fh)
    # signed coefficients (BASELINE config 2).  The reference rejects negative
    # coefficients (pack.py:44-46), so the expected product is the reference's
    # own signed schoolbook convolution (oracle.uni_schoolbook over ring_z,
    # oracle.py:58-69), cross-checked against the bias lift through the
    # reference ks*_mul (f' = f + 2^31, b = 32).
    import operator
    uni = K.uni_schoolbook(Z, operator.mul)
    scases = []
    for i in range(24):
        lf = rng.choice([1, 2, 3, 5, 16, 64, 100, 257])
        lg = lf if i % 2 == 0 else rng.choice([1, 2, 7, 64, 128])
        f = [rng.randrange(-2**31, 2**31) for _ in range(lf)]
        g = [rng.randrange(-2**31, 2**31) for _ in range(lg)]
        if i == 0:
            f, g = [-2**31] * 8, [-2**31] * 8     # extreme: |h| = 8 * 2^62
            lf = lg = 8
        want = uni(f, g)
        bias = 1 << 31
        F = K.CoeffVec(tuple(c + bias for c in f), 32)
        G = K.CoeffVec(tuple(c + bias for c in g), 32)
        for fn in VARIANTS.values():
            hl = fn(F, G).coeffs
            fix = []
            for k in range(lf + lg - 1):
                i0, i1 = max(0, k - lg + 1), min(k, lf - 1)
                j0, j1 = max(0, k - lf + 1), min(k, lg - 1)
                sf = sum(c + bias for c in f[i0:i1 + 1])
                sg = sum(c + bias for c in g[j0:j1 + 1])
                fix.append(hl[k] - bias * (sf + sg) + bias * bias * (i1 - i0 + 1))
            assert fix == want
        scases.append({"f": f, "g": g, "h": [str(v) for v in want]})
    with gzip.open(os.path.join(HERE, "signed_golden.json.gz"), "wt") as fh:
        json.dump(scases, fh)
    print("cases:", len(cases), "packs:", len(packs), "recs:", len(recs), "bivar:", len(bcases))


if __name__ == "__main__":
    main()
