"""Drop-in integer Kronecker substitution entry points, computed on the GPU.

Mirrors pkg/src/kronmul/ksint.py: same names, signatures, return types and
exceptions; every product runs through libkmx.so (pack -> multiply ->
finish -> reconstruct kernels on sm_100a).  There is no CPU fallback.

  derive_params          ksint.py:82-98 (host scalars)
  ks1_mul .. ks4_mul     ksint.py:219-348   (kmx_ks_mul_host)
  reconstruct_overlapped ksint.py:182-195   (kmx_reconstruct_host)
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import ReconstructionError, check, lib
from .kstypes import DEFAULT_MUL_CONFIG, CoeffVec, KsParams, MulConfig, MulStats, OverlapDigits
from .words import ints_to_words, words_to_ints

__all__ = ["KsParams", "OverlapDigits", "ReconstructionError", "derive_params", "ks1_mul",
           "ks2_mul", "ks3_mul", "ks4_mul", "reconstruct_overlapped"]


def derive_params(len_f: int, len_g: int, coeff_bits: int) -> KsParams:
    """Chunk widths for inputs of the given lengths and bit bound
    (ksint.py:82-98).  Host scalars, so computed here for any size; the
    kernels take the same widths from kmx_ks_params (tests/test_abi.py
    checks that the two agree)."""
    if len_f < 1 or len_g < 1:
        raise ValueError("polynomial lengths must be >= 1")
    if coeff_bits < 1:
        raise ValueError("coefficient bit bound must be >= 1")
    e = _e(len_f, len_g)
    full = 2 * coeff_bits + e
    return KsParams(len_f, len_g, coeff_bits, e, full, coeff_bits + (e + 1) // 2, (full + 3) // 4)


def _nlimbs64(x: int) -> int:
    return (x.bit_length() + 63) // 64


def _mul_count(x: int, y: int, config: MulConfig) -> int:
    """The 64-bit word products ``bignat.mul(x, y, stats, config)`` counts
    (bignat.py:323-371): the classical product of an m x n operand pair counts
    m*n; above ``karatsuba_threshold`` the three-product recursion splits at
    half the longer operand and counts its leaves.  Only operand LENGTHS are
    followed here (splits and the two sums per node) -- no product is formed
    on the host."""
    xl, yl = _nlimbs64(x), _nlimbs64(y)
    thr = config.karatsuba_threshold
    if config.classical_only or xl <= thr or yl <= thr:
        return xl * yl
    half = (max(xl, yl) + 1) // 2
    shift = 64 * half
    mask = (1 << shift) - 1
    x0, x1, y0, y1 = x & mask, x >> shift, y & mask, y >> shift
    # (inside the recursion the reference tests only the threshold, bignat.py:346-347)
    rec = MulConfig(karatsuba_threshold=thr, classical_only=False)
    return _mul_count(x0, y0, rec) + _mul_count(x1, y1, rec) + _mul_count(x0 + x1, y0 + y1, rec)


def _stats_count(variant: int, f: CoeffVec, g: CoeffVec, config: MulConfig) -> int:
    """MulStats.limb_products of the reference's ksN_mul(f, g, config=config)
    (ksint.py:219-348): the operands are the GPU packs (K1), the count follows
    the reference's dispatch."""
    from .pack import pack, pack_negated, pack_negated_reversed, pack_reversed
    p = derive_params(len(f.coeffs), len(g.coeffs), max(f.width_bound_bits, g.width_bound_bits))
    if variant == 4:
        w = 2 * p.width_quarter
        if not p.coeff_product_bound() < (1 << w) * ((1 << w) - 1):
            variant = 1  # ksint.py:301-302
        elif p.out_len == 1:
            return _mul_count(f.coeffs[0], g.coeffs[0], config)
    if variant == 1:
        n, kinds = p.width_full, (pack,)
    elif variant == 2:
        n, kinds = p.width_half, (pack, pack_reversed)
    elif variant == 3:
        n, kinds = p.width_half, (pack, pack_negated)
    else:
        n, kinds = p.width_quarter, (pack, pack_negated, pack_reversed, pack_negated_reversed)
    return sum(_mul_count(abs(fn(f, n)), abs(fn(g, n)), config) for fn in kinds)


def _ks(variant: int, f: CoeffVec, g: CoeffVec, stats: MulStats | None, config: MulConfig | None = None) -> CoeffVec:
    b = max(f.width_bound_bits, g.width_bound_bits)
    words = (b + 31) // 32
    lf, lg = len(f.coeffs), len(g.coeffs)
    fw = ints_to_words(f.coeffs, words)
    gw = ints_to_words(g.coeffs, words)
    ow = lib().kmx_ks_out_words(lf, lg, b, 0)
    if ow < 0:
        check(ow, f"ks{variant}_mul")
    h = np.zeros((lf + lg - 1, ow), dtype=np.uint32)
    lp = ctypes.c_uint64(0)
    rc = lib().kmx_ks_mul_host(variant, 1, lf, lg, b, _lib.ptr(fw), _lib.ptr(gw), words,
                               _lib.ptr(h), ow, 0, ctypes.byref(lp) if stats is not None else None)
    check(rc, f"ks{variant}_mul")
    if stats is not None:
        cfg = config if config is not None else DEFAULT_MUL_CONFIG
        if cfg.classical_only:
            stats.limb_products += int(lp.value)  # counted on the device from K1's bit lengths
        else:
            stats.limb_products += _stats_count(variant, f, g, cfg)
    return CoeffVec(tuple(words_to_ints(h)), 2 * b + _e(lf, lg))


def _e(lf: int, lg: int) -> int:
    return (min(lf, lg) - 1).bit_length()


def ks1_mul(f: CoeffVec, g: CoeffVec, *, stats: MulStats | None = None,
            config: MulConfig | None = None) -> CoeffVec:
    """Standard substitution: one full-width product (ksint.py:219-226)."""
    return _ks(1, f, g, stats, config)


def ks2_mul(f: CoeffVec, g: CoeffVec, *, stats: MulStats | None = None,
            config: MulConfig | None = None, parallel: bool = False) -> CoeffVec:
    """Reciprocal variant: forward and reversed half-width products, carry
    reconstruction (ksint.py:229-247).  ``parallel`` is accepted for
    signature compatibility: the sub-products always run concurrently on the
    GPU, with bit-identical results."""
    return _ks(2, f, g, stats, config)


def ks3_mul(f: CoeffVec, g: CoeffVec, *, stats: MulStats | None = None,
            config: MulConfig | None = None, parallel: bool = False) -> CoeffVec:
    """Negated variant: products at +-2^N, half-sum / half-difference
    (ksint.py:257-279)."""
    return _ks(3, f, g, stats, config)


def ks4_mul(f: CoeffVec, g: CoeffVec, *, stats: MulStats | None = None,
            config: MulConfig | None = None, parallel: bool = False) -> CoeffVec:
    """Four-point variant: quarter-width products at +-2^N and +-2^-N, even/odd
    split, two overlap reconstructions; KS1 fallback when the bound is not
    certified (ksint.py:289-348)."""
    return _ks(4, f, g, stats, config)


def reconstruct_overlapped(d: OverlapDigits, *, with_carries: bool = False):
    """Recover the coefficients behind two overlapped packings
    (ksint.py:182-195), on the GPU."""
    w = d.width_bits
    count = d.coeff_count
    dw = (w + 31) // 32
    fw = ints_to_words(d.forward_digits, dw)
    rw = ints_to_words(d.reversed_digits, dw)
    hw = (2 * w + 31) // 32
    h = np.zeros((count, hw), dtype=np.uint32)
    car = np.zeros(2 * count + 1, dtype=np.uint8) if with_carries else None
    rc = lib().kmx_reconstruct_host(1, count, w, _lib.ptr(fw), _lib.ptr(rw), dw, _lib.ptr(h), hw,
                                    _lib.ptr(car) if car is not None else None)
    check(rc, "reconstruct_overlapped")
    out = CoeffVec(tuple(words_to_ints(h)), 2 * w)
    if with_carries:
        return out, [int(x) for x in car[:count + 1]], [int(x) for x in car[count + 1:]]
    return out
