"""Drop-in evaluation functions of kronmul.pack, computed by K1 on the GPU.

Mirrors pkg/src/kronmul/pack.py:79-110: ``pack`` (value at 2^w),
``pack_reversed`` (at 2^-w, normalized), ``pack_negated`` (at -2^w) and
``pack_negated_reversed`` (at -2^-w, normalized; sign flipped for even
lengths), with the same width check (pack.py:55-59 -> ValueError).  The
reference returns a BigNat / SignedBig; these return the Python int those
objects convert to (``int(BigNat)``, ``SignedBig.value``).  ``pack_batch``
is the batched form over a [batch, len, words] array (one K1 launch).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, lib
from .kstypes import CoeffVec
from .words import ints_to_words, words_to_ints

__all__ = ["pack", "pack_reversed", "pack_negated", "pack_negated_reversed", "pack_batch"]

KIND = {"pack": 0, "pack_negated": 1, "pack_reversed": 2, "pack_negated_reversed": 3}


def pack_batch(kind: int, coeffs: np.ndarray, width_bits: int, coeff_bits: int):
    """coeffs [batch, len, words] uint32 -> (|values| [batch, limbs] uint32
    (limbs = kmx_pack_limbs rounded up to a multiple of 4),
    meta [batch, 2] = sign, bit length) through kmx_pack_host."""
    coeffs = np.ascontiguousarray(coeffs, dtype=np.uint32)
    batch, length, words = coeffs.shape
    m = lib().kmx_pack_limbs(length, width_bits, coeff_bits)
    if m < 0:
        check(m, "pack")
    out = np.zeros((batch, (m + 3) & ~3), dtype=np.uint32)  # K1 stores 16-byte limb quads
    meta = np.zeros((batch, 2), dtype=np.uint32)
    check(lib().kmx_pack_host(kind, batch, length, width_bits, coeff_bits, _lib.ptr(coeffs), words,
                              _lib.ptr(out), out.shape[1], _lib.ptr(meta)), "pack")
    return out, meta


def _one(kind: int, v: CoeffVec, width_bits: int) -> int:
    if 2 * width_bits < v.width_bound_bits:
        raise ValueError(f"chunk width {width_bits} below half the coefficient bound {v.width_bound_bits}")
    b = v.width_bound_bits
    words = (b + 31) // 32
    out, meta = pack_batch(kind, ints_to_words(v.coeffs, words)[None], width_bits, b)
    mag = words_to_ints(out[0][None, :])[0]
    return -mag if meta[0, 0] else mag


def pack(v: CoeffVec, width_bits: int) -> int:
    """Value of v at 2**width_bits (pack.py:79-82)."""
    return _one(0, v, width_bits)


def pack_reversed(v: CoeffVec, width_bits: int) -> int:
    """Value of the reversed vector at 2**width_bits (pack.py:85-91)."""
    return _one(2, v, width_bits)


def pack_negated(v: CoeffVec, width_bits: int) -> int:
    """Value of v at -2**width_bits (pack.py:94-97)."""
    return _one(1, v, width_bits)


def pack_negated_reversed(v: CoeffVec, width_bits: int) -> int:
    """Value of v at -2**(-width_bits), normalized (pack.py:100-110)."""
    return _one(3, v, width_bits)
