"""Command-line front end on the GPU path (mirrors kronmul/cli.py).

  python -m paper_0712_4046_b200 mul F G [-o H] [--modulus N] [--variant ks1..ks4|auto]
  python -m paper_0712_4046_b200 bench [--modulus-bits B] [--degrees lo:hi:log|lo:hi:+step]
                                       [--variants ks1,ks2,ks3,ks4] [--reps R] [--seed S]
                                       [--count-ops] [--batch P] [-o CSV]

Same polynomial file format (cli.py:62-96: decimal modulus, decimal length L,
then L coefficients, constant term first) and the same bench CSV schema
(cli.py:32, :157-171, :192-245), so GPU and CPU rows are directly comparable:
the header line is the reference's CSV_HEADER unchanged, and the device, the
batch and the timing method go into the leading ``#`` comment line.

``wall_ns_median`` is the median wall time of one product through the public
host API (``mod_mul``: host buffers, copies and the kernels inside the timed
call, as the reference times ``mod_mul``); with ``--batch P`` one call
multiplies P independent pairs (``mod_mul_host``) and the column is the time
per product.  ``limb_products`` (``--count-ops``) is the reference's classical
count (``MulStats``), reported by the pack kernel.
"""
from __future__ import annotations

import argparse
import random
import statistics
import sys
import time
from dataclasses import dataclass

import numpy as np

from .kstypes import MulStats
from .modpoly import ModPoly, Variant, mod_mul, mod_mul_host

CSV_HEADER = "degree,length,modulus_bits,variant,wall_ns_median,limb_products,ratio_vs_ks1"


class CommandError(Exception):
    """A user-facing failure; the message goes to stderr, exit status 1."""


# --- polynomial files (cli.py:62-96) -------------------------------------------

def read_poly_file(path: str) -> ModPoly:
    try:
        with open(path, "r", encoding="ascii") as fh:
            tokens = fh.read().split()
    except OSError as exc:
        raise CommandError(f"cannot read {path}: {exc}")
    if len(tokens) < 2:
        raise CommandError(f"{path}: expected modulus and length")
    try:
        modulus, length = int(tokens[0]), int(tokens[1])
        coeffs = [int(t) for t in tokens[2:]]
    except ValueError as exc:
        raise CommandError(f"{path}: {exc}")
    if length != len(coeffs):
        raise CommandError(f"{path}: declared length {length} but found {len(coeffs)} coefficients")
    try:
        return ModPoly(tuple(coeffs), modulus)
    except ValueError as exc:
        raise CommandError(f"{path}: {exc}")


def format_poly(p: ModPoly) -> str:
    return "{}\n{}\n{}\n".format(p.modulus, len(p.coeffs), " ".join(str(c) for c in p.coeffs))


def write_poly_file(path: str, p: ModPoly) -> None:
    try:
        with open(path, "w", encoding="ascii") as fh:
            fh.write(format_poly(p))
    except OSError as exc:
        raise CommandError(f"cannot write {path}: {exc}")


def _parse_variant(name: str) -> Variant:
    try:
        return Variant(name.lower())
    except ValueError:
        raise CommandError(f"unknown variant {name!r}")


def cmd_mul(args) -> int:
    f = read_poly_file(args.poly_f)
    g = read_poly_file(args.poly_g)
    if f.modulus != g.modulus:
        raise CommandError(f"modulus mismatch: {f.modulus} vs {g.modulus}")
    if args.modulus is not None and args.modulus != f.modulus:
        raise CommandError(f"--modulus {args.modulus} does not match file modulus {f.modulus}")
    product = mod_mul(f, g, _parse_variant(args.variant))
    if args.output:
        write_poly_file(args.output, product)
    else:
        sys.stdout.write(format_poly(product))
    return 0


# --- bench (cli.py:123-272) ------------------------------------------------------

def parse_degree_grid(grid: str) -> list[int]:
    """``lo:hi:log`` (about 20 log-spaced points) or ``lo:hi:+step``."""
    parts = grid.split(":")
    if len(parts) != 3:
        raise CommandError(f"invalid degree grid {grid!r}")
    try:
        lo, hi = int(parts[0]), int(parts[1])
    except ValueError:
        raise CommandError(f"invalid degree grid {grid!r}")
    if lo < 1 or hi < lo:
        raise CommandError(f"invalid degree range {lo}:{hi}")
    if parts[2] == "log":
        return sorted({round(lo * (hi / lo) ** (i / 19)) for i in range(20)})
    if parts[2].startswith("+"):
        try:
            step = int(parts[2][1:])
        except ValueError:
            raise CommandError(f"invalid degree step {parts[2]!r}")
        if step < 1:
            raise CommandError("degree step must be >= 1")
        return list(range(lo, hi + 1, step))
    raise CommandError(f"invalid degree grid {grid!r}")


@dataclass
class BenchRow:
    degree: int
    length: int
    modulus_bits: int
    variant: str
    wall_ns_median: int
    limb_products: int | None
    ratio_vs_ks1: float | None

    def csv(self) -> str:
        ops = "" if self.limb_products is None else str(self.limb_products)
        ratio = "" if self.ratio_vs_ks1 is None else f"{self.ratio_vs_ks1:.4f}"
        return (f"{self.degree},{self.length},{self.modulus_bits},"
                f"{self.variant},{self.wall_ns_median},{ops},{ratio}")


def _median_call_ns(fn, reps: int) -> int:
    """cli.py:174-189: discard a warm-up, batch fast calls to >= ~2 ms."""
    fn()
    t0 = time.perf_counter_ns()
    fn()
    single = max(1, time.perf_counter_ns() - t0)
    iters = min(256, 2_000_000 // single + 1) if single < 2_000_000 else 1
    samples = []
    for _ in range(reps):
        t0 = time.perf_counter_ns()
        for _ in range(iters):
            fn()
        samples.append((time.perf_counter_ns() - t0) // iters)
    return int(statistics.median(samples))


def _device_name() -> str:
    try:
        import torch
        return torch.cuda.get_device_name(0).replace(",", " ")
    except Exception:
        return "cuda"


def run_bench(degrees, modulus_bits: int, variants, reps: int, seed: int, count_ops: bool = False,
              batch: int = 1):
    """Time every (degree, variant) cell on shared random inputs
    (cli.py:192-245).  Returns (comment_lines, rows)."""
    if reps < 1:
        raise CommandError("reps must be >= 1")
    if batch < 1:
        raise CommandError("batch must be >= 1")
    if modulus_bits < 1 or modulus_bits > 64:
        raise CommandError("modulus bits must be in [1, 64]")
    variants = [v if isinstance(v, Variant) else _parse_variant(v) for v in variants]
    if any(v is Variant.AUTO for v in variants):
        raise CommandError("bench variants must be explicit (no auto)")
    rng = random.Random(seed)
    modulus = max(2, rng.randrange(1 << (modulus_bits - 1), 1 << modulus_bits) if modulus_bits > 1 else 2)
    comments = [f"# seed={seed} modulus={modulus} parallel=False classical_only={count_ops} "
                f"karatsuba_threshold=none device={_device_name()} batch={batch} "
                f"timing=host-api-wall-per-product"]
    num = {Variant.KS1: 1, Variant.KS2: 2, Variant.KS3: 3, Variant.KS4: 4}
    rows: list[BenchRow] = []
    for degree in degrees:
        length = degree + 1
        f = ModPoly(tuple(rng.randrange(modulus) for _ in range(length)), modulus)
        g = ModPoly(tuple(rng.randrange(modulus) for _ in range(length)), modulus)
        fb = np.tile(np.array(f.coeffs, dtype=np.uint64), (batch, 1))
        gb = np.tile(np.array(g.coeffs, dtype=np.uint64), (batch, 1))
        cell: dict[Variant, BenchRow] = {}
        for variant in variants:
            if batch == 1:
                def call(v=variant):
                    return mod_mul(f, g, v)
            else:
                out = np.empty((batch, 2 * length - 1), dtype=np.uint64)

                def call(v=variant, out=out):
                    return mod_mul_host(num[v], fb, gb, modulus, out=out)
            median = _median_call_ns(call, reps) // batch
            ops = None
            if count_ops:
                stats = MulStats()
                mod_mul(f, g, variant, stats=stats)
                ops = stats.limb_products
            row = BenchRow(degree, length, modulus_bits, variant.value, max(1, median), ops, None)
            cell[variant] = row
            rows.append(row)
        base = cell.get(Variant.KS1)
        if base is not None and base.wall_ns_median > 0:
            for row in cell.values():
                row.ratio_vs_ks1 = row.wall_ns_median / base.wall_ns_median
    return comments, rows


def render_csv(comments, rows) -> str:
    lines = list(comments)
    lines.append(CSV_HEADER)
    lines.extend(row.csv() for row in rows)
    return "\n".join(lines) + "\n"


def cmd_bench(args) -> int:
    degrees = parse_degree_grid(args.degrees)
    variants = [v.strip() for v in args.variants.split(",") if v.strip()]
    if not variants:
        raise CommandError("no variants requested")
    comments, rows = run_bench(degrees, args.modulus_bits, variants, args.reps, args.seed,
                               count_ops=args.count_ops, batch=args.batch)
    text = render_csv(comments, rows)
    if args.output:
        try:
            with open(args.output, "w", encoding="ascii") as fh:
                fh.write(text)
        except OSError as exc:
            raise CommandError(f"cannot write {args.output}: {exc}")
    else:
        sys.stdout.write(text)
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_0712_4046_b200",
                                     description="Polynomial multiplication over Z/nZ via multipoint "
                                                 "Kronecker substitution on B200.")
    sub = parser.add_subparsers(dest="command", required=True)
    p_mul = sub.add_parser("mul", help="multiply two polynomial files")
    p_mul.add_argument("poly_f")
    p_mul.add_argument("poly_g")
    p_mul.add_argument("-o", "--output", help="output file (default stdout)")
    p_mul.add_argument("--modulus", type=int, help="expected modulus; must match the input files")
    p_mul.add_argument("--variant", default="auto", choices=["ks1", "ks2", "ks3", "ks4", "auto"])
    p_mul.add_argument("--parallel", action="store_true", help="accepted for compatibility (no effect)")
    p_mul.set_defaults(func=cmd_mul)
    p_bench = sub.add_parser("bench", help="benchmark variants to CSV")
    p_bench.add_argument("--modulus-bits", type=int, default=48)
    p_bench.add_argument("--degrees", default="100:5000:log", help="grid: lo:hi:log or lo:hi:+step")
    p_bench.add_argument("--variants", default="ks1,ks2,ks3,ks4")
    p_bench.add_argument("--reps", type=int, default=5, help="timed repetitions per cell (median taken)")
    p_bench.add_argument("--seed", type=int, default=1)
    p_bench.add_argument("--count-ops", action="store_true", help="also record the classical limb-product counts")
    p_bench.add_argument("--batch", type=int, default=1, help="independent pairs per call (time per product)")
    p_bench.add_argument("--parallel", action="store_true", help="accepted for compatibility (no effect)")
    p_bench.add_argument("-o", "--output", help="CSV file (default stdout)")
    p_bench.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except CommandError as exc:
        print(f"paper_0712_4046_b200: {exc}", file=sys.stderr)
        return 1
