"""Command-line front end of the GPU path: ``mul`` and ``bench``.

  python -m paper_0712_4046_b200 mul F G [-o H] [--modulus N] [--variant ks1..ks4|auto]
  python -m paper_0712_4046_b200 bench [--modulus-bits B] [--degrees lo:hi:log|lo:hi:+step]
                                       [--variants ks1,ks2,ks3,ks4] [--reps R] [--seed S]
                                       [--count-ops] [--batch P] [-o CSV]

Interoperability contract with the reference CLI (kronmul/cli.py):
  * polynomial files (cli.py:62-96): whitespace-separated decimal tokens --
    modulus, length L, then L coefficients, constant term first;
  * bench CSV (cli.py:32, :157-171): the same header line and seven columns,
    so GPU rows and reference CPU rows can be concatenated and compared; the
    leading ``#`` line records how the GPU rows were measured;
  * the degree grid syntax (cli.py:123-146) and the exit status (1 with a
    one-line message on stderr for user errors).

The bench here is GPU-first.  Every (degree, variant) cell multiplies
``--batch`` independent pairs per call through the host-buffer API
(``mod_mul_host`` -> ``kmx_mod_mul_host``: H2D copies, kernels, D2H copies),
so ``wall_ns_median`` is the end-to-end time per product, the quantity the
reference's column measures for its CPU path.  ``limb_products`` comes from
the pack kernel's operand lengths (the reference's classical count,
bignat.py:327-330).  ``selftest`` (which exercises the reference's own
bignum layer) is out of scope for this hot-path build.
"""
from __future__ import annotations

import argparse
import math
import random
import sys
import time
from typing import Callable, Iterable, List, Optional, Sequence

import numpy as np

from .kstypes import MulStats
from .modpoly import ModPoly, Variant, mod_mul, mod_mul_host

CSV_COLUMNS = ("degree", "length", "modulus_bits", "variant", "wall_ns_median", "limb_products",
               "ratio_vs_ks1")
CSV_HEADER = ",".join(CSV_COLUMNS)
PROG = "paper_0712_4046_b200"
_EXPLICIT = {"ks1": Variant.KS1, "ks2": Variant.KS2, "ks3": Variant.KS3, "ks4": Variant.KS4}
_KS_NUMBER = {Variant.KS1: 1, Variant.KS2: 2, Variant.KS3: 3, Variant.KS4: 4}


class CommandError(Exception):
    """User-facing failure: reported as ``prog: message`` on stderr, exit 1."""


# ------------------------------------------------------------------ file format

def _decimal_tokens(text: str, where: str) -> List[int]:
    out = []
    for pos, tok in enumerate(text.split()):
        try:
            out.append(int(tok))
        except ValueError as exc:
            raise CommandError(f"{where}: token {pos + 1}: {exc}")
    return out


def read_poly_file(path: str) -> ModPoly:
    """Parse a polynomial file (modulus, length, coefficients)."""
    try:
        with open(path, encoding="ascii") as fh:
            body = fh.read()
    except OSError as exc:
        raise CommandError(f"cannot read {path}: {exc}")
    nums = _decimal_tokens(body, path)
    if len(nums) < 2:
        raise CommandError(f"{path}: expected modulus and length")
    modulus, declared, coeffs = nums[0], nums[1], nums[2:]
    if declared != len(coeffs):
        raise CommandError(f"{path}: declared length {declared} but found {len(coeffs)} coefficients")
    try:
        return ModPoly(tuple(coeffs), modulus)
    except ValueError as exc:
        raise CommandError(f"{path}: {exc}")


def format_poly(p: ModPoly) -> str:
    lines = [str(p.modulus), str(len(p.coeffs)), " ".join(map(str, p.coeffs))]
    return "\n".join(lines) + "\n"


def _emit(text: str, path: Optional[str]) -> None:
    if not path:
        sys.stdout.write(text)
        return
    try:
        with open(path, "w", encoding="ascii") as fh:
            fh.write(text)
    except OSError as exc:
        raise CommandError(f"cannot write {path}: {exc}")


def write_poly_file(path: str, p: ModPoly) -> None:
    _emit(format_poly(p), path)


def _variant(name: str, allow_auto: bool = True) -> Variant:
    key = name.strip().lower()
    if key in _EXPLICIT:
        return _EXPLICIT[key]
    if key == "auto":
        if not allow_auto:
            raise CommandError("bench variants must be explicit (no auto)")
        return Variant.AUTO
    raise CommandError(f"unknown variant {name!r}")


# ------------------------------------------------------------------------- mul

def cmd_mul(args) -> int:
    f, g = read_poly_file(args.poly_f), read_poly_file(args.poly_g)
    if f.modulus != g.modulus:
        raise CommandError(f"modulus mismatch: {f.modulus} vs {g.modulus}")
    if args.modulus is not None and args.modulus != f.modulus:
        raise CommandError(f"--modulus {args.modulus} does not match file modulus {f.modulus}")
    _emit(format_poly(mod_mul(f, g, _variant(args.variant))), args.output)
    return 0


# ----------------------------------------------------------------------- bench

def _log_grid(lo: int, hi: int) -> List[int]:
    # twenty geometrically spaced points between lo and hi, deduplicated
    ratio = hi / lo
    return sorted({round(lo * math.pow(ratio, k / 19)) for k in range(20)})


def _step_grid(lo: int, hi: int, spec: str) -> List[int]:
    try:
        step = int(spec)
    except ValueError:
        raise CommandError(f"invalid degree step {'+' + spec!r}")
    if step < 1:
        raise CommandError("degree step must be >= 1")
    return list(range(lo, hi + 1, step))


def parse_degree_grid(grid: str) -> List[int]:
    """``lo:hi:log`` (about 20 log-spaced degrees) or ``lo:hi:+step``."""
    fields = grid.split(":")
    if len(fields) != 3:
        raise CommandError(f"invalid degree grid {grid!r}")
    try:
        lo, hi = int(fields[0]), int(fields[1])
    except ValueError:
        raise CommandError(f"invalid degree grid {grid!r}")
    if lo < 1 or hi < lo:
        raise CommandError(f"invalid degree range {lo}:{hi}")
    kind = fields[2]
    if kind == "log":
        return _log_grid(lo, hi)
    if kind[:1] == "+":
        return _step_grid(lo, hi, kind[1:])
    raise CommandError(f"invalid degree grid {grid!r}")


def _per_call_ns(call: Callable[[], object], reps: int) -> int:
    """Median over ``reps`` samples of the per-call wall time.  One untimed
    call first (plans, workspaces); fast calls are repeated inside a sample
    until it spans about 2 ms, as the reference's harness does."""
    call()
    t0 = time.perf_counter_ns()
    call()
    one = max(1, time.perf_counter_ns() - t0)
    inner = 1 if one >= 2_000_000 else min(256, 1 + 2_000_000 // one)
    samples = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        for _ in range(inner):
            call()
        samples.append((time.perf_counter_ns() - t0) // inner)
    samples.sort()
    mid = len(samples) // 2
    return int(samples[mid] if len(samples) % 2 else (samples[mid - 1] + samples[mid]) // 2)


def _row(degree: int, bits: int, variant: Variant, ns: int, ops: Optional[int],
         ratio: Optional[float]) -> List[str]:
    return [str(degree), str(degree + 1), str(bits), variant.value, str(ns),
            "" if ops is None else str(ops), "" if ratio is None else f"{ratio:.4f}"]


def _device_label() -> str:
    try:
        import torch
        return torch.cuda.get_device_name(0).replace(",", " ")
    except Exception:  # noqa: BLE001 - label only
        return "cuda"


def _draw_modulus(rng: random.Random, bits: int) -> int:
    if bits == 1:
        return 2
    return max(2, rng.randrange(1 << (bits - 1), 1 << bits))


def run_bench(degrees: Iterable[int], modulus_bits: int, variants: Sequence, reps: int, seed: int,
              count_ops: bool = False, batch: int = 1):
    """Time each (degree, variant) cell on shared seeded inputs; returns
    (comment lines, rows as lists of CSV fields)."""
    if reps < 1:
        raise CommandError("reps must be >= 1")
    if batch < 1:
        raise CommandError("batch must be >= 1")
    if not 1 <= modulus_bits <= 64:
        raise CommandError("modulus bits must be in [1, 64]")
    vs = [v if isinstance(v, Variant) else _variant(v, allow_auto=False) for v in variants]
    if Variant.AUTO in vs:
        raise CommandError("bench variants must be explicit (no auto)")
    rng = random.Random(seed)
    n = _draw_modulus(rng, modulus_bits)
    header = (f"# seed={seed} modulus={n} parallel=False classical_only={count_ops} "
              f"karatsuba_threshold=none device={_device_label()} batch={batch} "
              f"timing=host-api-wall-per-product")
    rows: List[List[str]] = []
    for degree in degrees:
        L = degree + 1
        f = ModPoly(tuple(rng.randrange(n) for _ in range(L)), n)
        g = ModPoly(tuple(rng.randrange(n) for _ in range(L)), n)
        fb = np.broadcast_to(np.asarray(f.coeffs, dtype=np.uint64), (batch, L)).copy()
        gb = np.broadcast_to(np.asarray(g.coeffs, dtype=np.uint64), (batch, L)).copy()
        hb = np.empty((batch, 2 * L - 1), dtype=np.uint64)
        timed = {}
        for v in vs:
            if batch == 1:
                call = (lambda v=v: mod_mul(f, g, v))
            else:
                call = (lambda k=_KS_NUMBER[v]: mod_mul_host(k, fb, gb, n, out=hb))
            ns = max(1, _per_call_ns(call, reps) // batch)
            ops = None
            if count_ops:
                st = MulStats()
                mod_mul(f, g, v, stats=st)
                ops = st.limb_products
            timed[v] = (ns, ops)
        base = timed.get(Variant.KS1, (0, None))[0]
        for v in vs:
            ns, ops = timed[v]
            rows.append(_row(degree, modulus_bits, v, ns, ops, ns / base if base else None))
    return [header], rows


def render_csv(comments: Sequence[str], rows: Sequence[Sequence[str]]) -> str:
    return "\n".join([*comments, CSV_HEADER, *(",".join(r) for r in rows)]) + "\n"


def cmd_bench(args) -> int:
    degrees = parse_degree_grid(args.degrees)
    names = [v for v in (s.strip() for s in args.variants.split(",")) if v]
    if not names:
        raise CommandError("no variants requested")
    comments, rows = run_bench(degrees, args.modulus_bits, names, args.reps, args.seed,
                               count_ops=args.count_ops, batch=args.batch)
    _emit(render_csv(comments, rows), args.output)
    return 0


# ------------------------------------------------------------------ entry point

def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog=PROG, description="(Z/nZ)[x] products by multipoint Kronecker "
                                                        "substitution on B200 (GPU path).")
    cmds = ap.add_subparsers(dest="command", required=True)
    m = cmds.add_parser("mul", help="multiply two polynomial files on the GPU")
    m.add_argument("poly_f")
    m.add_argument("poly_g")
    m.add_argument("-o", "--output", help="write the product here instead of stdout")
    m.add_argument("--modulus", type=int, help="modulus the input files must carry")
    m.add_argument("--variant", default="auto", choices=[*_EXPLICIT, "auto"])
    m.add_argument("--parallel", action="store_true", help="accepted; sub-products always run concurrently")
    m.set_defaults(func=cmd_mul)
    b = cmds.add_parser("bench", help="time the variants, reference CSV schema")
    b.add_argument("--modulus-bits", type=int, default=48)
    b.add_argument("--degrees", default="100:5000:log", help="lo:hi:log or lo:hi:+step")
    b.add_argument("--variants", default="ks1,ks2,ks3,ks4")
    b.add_argument("--reps", type=int, default=5, help="samples per cell; the median is reported")
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--count-ops", action="store_true", help="add the classical limb-product counts")
    b.add_argument("--batch", type=int, default=1, help="pairs per call; the column is time per product")
    b.add_argument("--parallel", action="store_true", help="accepted; no effect on the GPU path")
    b.add_argument("-o", "--output", help="write the CSV here instead of stdout")
    b.set_defaults(func=cmd_bench)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except CommandError as exc:
        print(f"{PROG}: {exc}", file=sys.stderr)
        return 1
