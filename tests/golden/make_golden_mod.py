"""Generate (Z/nZ)[x] golden vectors from the REFERENCE package itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_mod.py

Imports ``kronmul`` from /root/reference/pkg/src (read-only) and records, for
seeded inputs, the exact outputs of ``kronmul.modpoly.mod_mul`` for every
explicit variant (modpoly.py:95-115), cross-checked against the reference's
``oracle.schoolbook_mod`` (oracle.py:30-40), plus the classical-mode
``MulStats.limb_products`` counts and the ``choose_variant`` table
(modpoly.py:79-92).  The GPU box never reads /root/reference.
"""
import gzip
import json
import os
import random
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import kronmul as K  # noqa: E402
from kronmul.bignat import MulConfig, MulStats  # noqa: E402
from kronmul.modpoly import ModPoly, Variant, choose_variant, mod_mul  # noqa: E402
from kronmul.oracle import schoolbook_mod  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
EXPLICIT = [Variant.KS1, Variant.KS2, Variant.KS3, Variant.KS4]


def case(f, g, n, tag, stats=False):
    F, G = ModPoly(tuple(f), n), ModPoly(tuple(g), n)
    want = mod_mul(F, G, Variant.KS1).coeffs
    for v in EXPLICIT + [Variant.AUTO]:
        assert mod_mul(F, G, v).coeffs == want, (tag, v)
    if len(f) * len(g) <= 40000:
        assert schoolbook_mod(F, G).coeffs == want, tag
    c = {"tag": tag, "n": str(n), "f": [str(x) for x in f], "g": [str(x) for x in g],
         "h": [str(x) for x in want]}
    if stats:
        counts = {}
        for v in EXPLICIT:
            s = MulStats()
            mod_mul(F, G, v, stats=s, config=MulConfig(classical_only=True))
            counts[v.value] = s.limb_products
        c["limb_products_classical"] = counts
    return c


def main():
    rng = random.Random(20261020)
    cases = [case([274, 610, 887, 621], [553, 298, 424, 790], 1000003, "worked_example"),
             case([1], [1], 2, "mod_two")]
    # tests/test_modpoly.py:47-60 shapes: bits 2, 4, 48, lengths < 60
    for bits in (2, 4, 48):
        for i in range(20):
            n = rng.randrange(max(2, 1 << (bits - 1)), 1 << bits)
            f = [rng.randrange(n) for _ in range(rng.randrange(1, 60))]
            g = [rng.randrange(n) for _ in range(rng.randrange(1, 60))]
            cases.append(case(f, g, n, f"random_b{bits}_{i}"))
    # even moduli (tests/test_modpoly.py:63-70) and word-size extremes
    for n in (2, 16, 2**48, 2**63, 2**64 - 59, 2**64 - 1, 3, 2**32 - 5, 2**32 + 15):
        f = [rng.randrange(n) for _ in range(20)]
        g = [rng.randrange(n) for _ in range(20)]
        cases.append(case(f, g, n, f"modulus_{n}"))
        cases.append(case([n - 1] * 33, [n - 1] * 17, n, f"allmax_{n}"))
    # the paper's section-4 experiment sizes: 4-bit and 48-bit moduli at longer lengths
    for n, L in ((13, 1000), ((1 << 48) - 59, 1000), ((1 << 48) - 59, 257), (11, 4096)):
        f = [rng.randrange(n) for _ in range(L)]
        g = [rng.randrange(n) for _ in range(L)]
        cases.append(case(f, g, n, f"paper_n{n}_L{L}"))
    # tests/test_modpoly.py:89-106: classical-mode limb-product counts
    f = [rng.randrange((1 << 48) - 59) for _ in range(128)]
    g = [rng.randrange((1 << 48) - 59) for _ in range(128)]
    cases.append(case(f, g, (1 << 48) - 59, "dispatch_counts", stats=True))
    table = [[L, bits, choose_variant(L, bits).value]
             for L in (1, 2, 16, 47, 48, 49, 100, 511, 512, 513, 1000, 4096) for bits in (1, 4, 7, 48, 64)]
    with gzip.open(os.path.join(HERE, "mod_golden.json.gz"), "wt") as fh:
        json.dump({"cases": cases, "choose_variant": table}, fh)
    print("mod cases:", len(cases))


if __name__ == "__main__":
    main()


def main_bivar():
    """bks_* over ring_zmod(n) with the reference's default UniMul
    (uni_schoolbook over the ring, bipoly.py:121-125)."""
    rng = random.Random(20261021)
    BV = {1: K.bks_standard, 2: K.bks_reciprocal, 3: K.bks_negated, 4: K.bks_four}
    cases = []
    for n in (7, 1009, 65537, (1 << 61) - 1, (1 << 64) - 59, 2, 16, 1 << 40):
        ring = K.ring_zmod(n)
        for i in range(6):
            lx, ly = rng.randrange(1, 9), rng.randrange(1, 9)
            if i == 0:
                lx = ly = 1
            f = [[rng.randrange(n) for _ in range(ly)] for _ in range(lx)]
            g = [[rng.randrange(n) for _ in range(ly)] for _ in range(lx)]
            F, G = K.BiPoly(tuple(map(tuple, f))), K.BiPoly(tuple(map(tuple, g)))
            outs = {}
            for v, fn in BV.items():
                try:
                    outs[v] = [list(r) for r in fn(F, G, ring).coeffs]
                except K.MissingHalveError:
                    outs[v] = None
            ok = [o for o in outs.values() if o is not None]
            assert all(o == ok[0] for o in ok)
            cases.append({"n": str(n), "f": [[str(c) for c in r] for r in f], "g": [[str(c) for c in r] for r in g],
                          "h": [[str(c) for c in r] for r in ok[0]],
                          "missing_halve": [v for v, o in outs.items() if o is None]})
    with gzip.open(os.path.join(HERE, "bivar_mod_golden.json.gz"), "wt") as fh:
        json.dump(cases, fh)
    print("bivar mod cases:", len(cases))


if __name__ == "__main__" and "--bivar" in sys.argv:
    main_bivar()
