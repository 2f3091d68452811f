"""Golden MulStats.limb_products values from the REFERENCE package.

Run in the builder container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_stats.py

For seeded inputs it records the word-product counts the reference reports
for ks1_mul .. ks4_mul (ksint.py:219-348 through bignat.mul, bignat.py:323-380)
under three dispatch policies: the default MulConfig (Karatsuba above 16
limbs), karatsuba_threshold=2, and classical_only.  The fixture is committed;
the GPU box never reads /root/reference.
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

HERE = os.path.dirname(os.path.abspath(__file__))
VARIANTS = {1: K.ks1_mul, 2: K.ks2_mul, 3: K.ks3_mul, 4: K.ks4_mul}
CONFIGS = {"default": None, "thr2": MulConfig(karatsuba_threshold=2), "classical": MulConfig(classical_only=True)}


def main():
    rng = random.Random(20260)
    shapes = [(1, 1, 8), (3, 2, 5), (16, 16, 8), (40, 17, 32), (64, 64, 64), (100, 37, 64), (128, 128, 32),
              (200, 200, 100), (256, 256, 64), (300, 5, 200), (512, 512, 16), (33, 33, 512), (700, 650, 40)]
    cases = []
    for lf, lg, b in shapes:
        for kind in ("rand", "max"):
            if kind == "rand":
                f = [rng.randrange(1 << b) for _ in range(lf)]
                g = [rng.randrange(1 << b) for _ in range(lg)]
            else:
                f = [(1 << b) - 1] * lf
                g = [(1 << b) - 1] * lg
            F, G = K.CoeffVec(tuple(f), b), K.CoeffVec(tuple(g), b)
            counts = {}
            for name, cfg in CONFIGS.items():
                row = []
                for v, fn in VARIANTS.items():
                    st = MulStats()
                    fn(F, G, stats=st, config=cfg)
                    row.append(st.limb_products)
                counts[name] = row
            cases.append({"b": b, "f": [format(x, "x") for x in f], "g": [format(x, "x") for x in g],
                          "counts": counts})
    with gzip.open(os.path.join(HERE, "stats_golden.json.gz"), "wt") as fh:
        json.dump(cases, fh)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
