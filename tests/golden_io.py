"""Loaders for the committed golden fixtures (generated from the reference by
tests/golden/make_golden.py)."""
import gzip
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt") as fh:
        return json.load(fh)


def _ints(hexlist):
    return [int(x, 16) for x in hexlist]


def ks_cases():
    out = []
    for c in _load("ks_golden.json.gz"):
        out.append((c["tag"], _ints(c["f"]), _ints(c["g"]), c["b"], _ints(c["h"])))
    return out


def pack_cases():
    out = []
    for c in _load("pack_golden.json.gz"):
        out.append((_ints(c["c"]), c["b"], c["w"], int(c["pack"]), int(c["rev"]),
                    int(c["neg"]), int(c["nrev"])))
    return out


def recon_cases():
    return [(_ints(c["fwd"]), _ints(c["rev"]), c["w"], _ints(c["h"]))
            for c in _load("recon_golden.json.gz")]


def bivar_cases():
    return [(c["tag"], c["f"], c["g"], c["h"]) for c in _load("bivar_golden.json.gz")]


def signed_cases():
    return [(c["f"], c["g"], [int(v) for v in c["h"]]) for c in _load("signed_golden.json.gz")]


def mod_golden():
    d = _load("mod_golden.json.gz")
    cases = []
    for c in d["cases"]:
        cases.append((c["tag"], [int(x) for x in c["f"]], [int(x) for x in c["g"]], int(c["n"]),
                      [int(x) for x in c["h"]], c.get("limb_products_classical")))
    return cases, [tuple(r) for r in d["choose_variant"]]


def bivar_mod_cases():
    out = []
    for c in _load("bivar_mod_golden.json.gz"):
        out.append((int(c["n"]), [[int(x) for x in r] for r in c["f"]], [[int(x) for x in r] for r in c["g"]],
                    [[int(x) for x in r] for r in c["h"]], c["missing_halve"]))
    return out


def stats_cases():
    """(f, g, b, {"default" | "thr2" | "classical": [ks1, ks2, ks3, ks4 counts]}) from the reference."""
    return [(_ints(c["f"]), _ints(c["g"]), c["b"], c["counts"]) for c in _load("stats_golden.json.gz")]
