"""Drop-in bivariate reductions R[x,y] -> R[x] over R = Z, on the GPU.

Mirrors pkg/src/kronmul/bipoly.py: BiPoly (:75-97), RingOps (:31-44),
ring_z (:53-56), ring_zmod (:59-72), MissingHalveError (:26-28) and
bks_standard / bks_reciprocal / bks_negated / bks_four (:177-278).

With ring_z() or ring_zmod(n) and the default univariate multiplier, the
whole reduction (evaluation, univariate products, half-sums and overlap
recovery) runs in libkmx.so: over Z through kmx_bks_mul (int32 coefficients,
int64 products) or, for wider coefficients, kmx_bks_wide_mul (any width: the
reduction over word-sized primes and CRT on the device); over Z/nZ through
kmx_bks_mod_mul (u64 residues; the univariate products go through the
integer KS path, kmx_mod_mul).  Custom univariate multipliers raise
NotImplementedError -- never a silent CPU path.
"""
from __future__ import annotations

import operator
from dataclasses import dataclass
from typing import Any, Callable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

__all__ = ["RingOps", "BiPoly", "MissingHalveError", "ring_z", "ring_zmod", "bks_standard",
           "bks_reciprocal", "bks_negated", "bks_four"]

UniMul = Callable[[Sequence[Any], Sequence[Any]], list]


class MissingHalveError(ValueError):
    """The ring has no exact halving, so this variant cannot run
    (bipoly.py:26-28)."""


@dataclass(frozen=True)
class RingOps:
    """Operation table of a commutative ring's additive structure
    (bipoly.py:31-44).  ``name`` identifies the rings the GPU path handles."""

    zero: Any
    add: Callable[[Any, Any], Any]
    sub: Callable[[Any, Any], Any]
    neg: Callable[[Any], Any]
    eq: Callable[[Any, Any], bool]
    halve: Optional[Callable[[Any], Any]] = None
    name: str = ""
    modulus: int = 0


def _halve_int(a: int) -> int:
    if a & 1:
        raise ValueError("halving an odd integer is not exact")
    return a >> 1


def ring_z() -> RingOps:
    """The integers (bipoly.py:53-56)."""
    return RingOps(zero=0, add=operator.add, sub=operator.sub, neg=operator.neg, eq=operator.eq,
                   halve=_halve_int, name="Z")


def ring_zmod(n: int) -> RingOps:
    """Integers mod n; halving exists only for odd n (bipoly.py:59-72)."""
    if n < 2:
        raise ValueError("modulus must be >= 2")
    halve = None
    if n % 2 == 1:
        inv2 = (n + 1) // 2
        halve = lambda a: (a * inv2) % n  # noqa: E731
    return RingOps(zero=0, add=lambda a, b: (a + b) % n, sub=lambda a, b: (a - b) % n,
                   neg=lambda a: (-a) % n, eq=operator.eq, halve=halve, name=f"Z/{n}", modulus=n)


@dataclass(frozen=True)
class BiPoly:
    """Dense bivariate polynomial: coeffs[i][j] is the coefficient of
    x**i * y**j (bipoly.py:75-97)."""

    coeffs: tuple

    def __post_init__(self):
        coeffs = tuple(tuple(row) for row in self.coeffs)
        object.__setattr__(self, "coeffs", coeffs)
        if not coeffs or not coeffs[0]:
            raise ValueError("both lengths must be >= 1")
        width = len(coeffs[0])
        if any(len(row) != width for row in coeffs):
            raise ValueError("coefficient array must be rectangular")

    @property
    def lx(self) -> int:
        return len(self.coeffs)

    @property
    def ly(self) -> int:
        return len(self.coeffs[0])


def _check_shapes(f: BiPoly, g: BiPoly) -> None:
    if f.lx != g.lx or f.ly != g.ly:
        raise ValueError("inputs must share both lengths")


def _bks(variant: int, f: BiPoly, g: BiPoly, ring: RingOps, mul: UniMul | None,
         needs_halve: bool) -> BiPoly:
    _check_shapes(f, g)
    if needs_halve and ring.halve is None:
        raise MissingHalveError("ring does not support exact halving")
    if mul is not None:
        raise NotImplementedError("custom univariate multipliers are not routed through the GPU path")
    lx, ly = f.lx, f.ly
    if ring.modulus:
        n = ring.modulus
        if n.bit_length() > 64:
            raise NotImplementedError("GPU Z/nZ path covers word-sized moduli (n < 2^64)")
        # ring elements as residues in [0, n) (the ring's own normalisation, bipoly.py:67-71)
        fu = np.array([[int(c) % n for c in row] for row in f.coeffs], dtype=np.uint64)
        gu = np.array([[int(c) % n for c in row] for row in g.coeffs], dtype=np.uint64)
        h = np.zeros((2 * lx - 1, 2 * ly - 1), dtype=np.uint64)
        rc = lib().kmx_bks_mod_mul_host(variant, 1, lx, ly, n, _lib.ptr(fu), _lib.ptr(gu), _lib.ptr(h))
        check(rc, "bks")
        return BiPoly(tuple(tuple(int(v) for v in row) for row in h))
    if ring.name != "Z":
        raise NotImplementedError("GPU bivariate path covers R = Z (ring_z) and R = Z/nZ (ring_zmod)")
    fa = np.asarray(f.coeffs, dtype=object)
    ga = np.asarray(g.coeffs, dtype=object)
    mx = max(max(abs(int(c)) for c in fa.reshape(-1)), max(abs(int(c)) for c in ga.reshape(-1)))
    cb = max(1, mx.bit_length())
    if cb <= 30:
        # int32 inputs, int64 univariate products (kmx_bks_mul) when the
        # accumulation bound holds; KMX_EINVAL otherwise -> the wide path
        f32 = np.ascontiguousarray(fa.astype(np.int64).astype(np.int32))
        g32 = np.ascontiguousarray(ga.astype(np.int64).astype(np.int32))
        h = np.zeros((2 * lx - 1, 2 * ly - 1), dtype=np.int64)
        rc = lib().kmx_bks_mul_host(variant, 1, lx, ly, cb, _lib.ptr(f32), _lib.ptr(g32), _lib.ptr(h))
        if rc != _lib.KMX_EINVAL:
            check(rc, "bks")
            return BiPoly(tuple(tuple(int(v) for v in row) for row in h))
    return _bks_wide(variant, f, g, lx, ly, cb)


def _bks_wide(variant: int, f: BiPoly, g: BiPoly, lx: int, ly: int, cb: int) -> BiPoly:
    """Any coefficient width over Z: kmx_bks_wide_mul (the reduction over
    word-sized primes, CRT on the device; two's-complement multiword I/O)."""
    from .words import ints_to_words, words_to_ints
    iw = (cb + 1 + 31) // 32
    ow = lib().kmx_bks_wide_out_words(lx, ly, cb)
    if ow < 0:
        check(ow, "bks")
    fw = ints_to_words([c for row in f.coeffs for c in row], iw, signed=True)
    gw = ints_to_words([c for row in g.coeffs for c in row], iw, signed=True)
    h = np.zeros(((2 * lx - 1) * (2 * ly - 1), ow), dtype=np.uint32)
    check(lib().kmx_bks_wide_mul_host(variant, 1, lx, ly, cb, _lib.ptr(fw), _lib.ptr(gw), iw, _lib.ptr(h), ow),
          "bks")
    vals = words_to_ints(h, signed=True)
    w2 = 2 * ly - 1
    return BiPoly(tuple(tuple(vals[i * w2:(i + 1) * w2]) for i in range(2 * lx - 1)))


def bks_standard(f: BiPoly, g: BiPoly, ring: RingOps, mul: UniMul | None = None) -> BiPoly:
    """One univariate product of length 2 Lx Ly - Lx - Ly + 1 (bipoly.py:177-188)."""
    return _bks(1, f, g, ring, mul, False)


def bks_reciprocal(f: BiPoly, g: BiPoly, ring: RingOps, mul: UniMul | None = None) -> BiPoly:
    """Two univariate products of length Lx Ly plus overlap recovery
    (bipoly.py:191-206)."""
    return _bks(2, f, g, ring, mul, False)


def bks_negated(f: BiPoly, g: BiPoly, ring: RingOps, mul: UniMul | None = None) -> BiPoly:
    """Two univariate products with alternating chunk signs, half-sum and
    half-difference (bipoly.py:209-232)."""
    return _bks(3, f, g, ring, mul, True)


def bks_four(f: BiPoly, g: BiPoly, ring: RingOps, mul: UniMul | None = None) -> BiPoly:
    """Four univariate products of length ceil(Lx/2)(Ly-1) + Lx
    (bipoly.py:235-278)."""
    return _bks(4, f, g, ring, mul, True)
