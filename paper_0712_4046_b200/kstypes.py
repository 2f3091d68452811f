"""Host-side value types mirroring the reference's public types for this path.

Same names, fields, validation and error behaviour as
  CoeffVec      pkg/src/kronmul/pack.py:25-52
  KsParams      pkg/src/kronmul/ksint.py:48-79
  OverlapDigits pkg/src/kronmul/ksint.py:101-134
  MulStats      pkg/src/kronmul/bignat.py:57-68
  MulConfig     pkg/src/kronmul/bignat.py:71-84
so tests written against the reference read the same against this package.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class CoeffVec:
    """Dense coefficient vector over the naturals, constant term first.

    Every coefficient satisfies 0 <= c < 2**width_bound_bits; the length is
    at least 1 (pack.py:25-52)."""

    coeffs: tuple
    width_bound_bits: int

    def __post_init__(self):
        coeffs = tuple(int(c) for c in self.coeffs)
        object.__setattr__(self, "coeffs", coeffs)
        if len(coeffs) < 1:
            raise ValueError("a coefficient vector has length >= 1")
        if self.width_bound_bits < 1:
            raise ValueError("width bound must be >= 1")
        bound = self.width_bound_bits
        for i, c in enumerate(coeffs):
            if c < 0 or c.bit_length() > bound:
                raise ValueError(f"coefficient {i} outside [0, 2**{bound})")

    def __len__(self) -> int:
        return len(self.coeffs)

    def reversed(self) -> "CoeffVec":
        return CoeffVec(self.coeffs[::-1], self.width_bound_bits)


@dataclass
class MulStats:
    """Counter of 64-bit word x word products (bignat.py:57-68), as the
    reference reports it for the given MulConfig: with ``classical_only`` the
    sum of limbs64(x) * limbs64(y) over the sub-products (bignat.py:327-330,
    counted on the device), otherwise the leaves of the reference's Karatsuba
    recursion (bignat.py:344-371; ksint._mul_count follows the operand
    lengths of the GPU-packed operands)."""

    limb_products: int = 0

    def reset(self) -> None:
        self.limb_products = 0


@dataclass(frozen=True)
class MulConfig:
    """Dispatch policy of the reference's bignum multiply (bignat.py:71-84).
    Results never depend on it (pkg/tests/test_ksint.py:93-112) and the GPU
    multiply kernels choose their own tiling; MulStats follows it."""

    karatsuba_threshold: int = 16
    classical_only: bool = False


DEFAULT_MUL_CONFIG = MulConfig()


@dataclass(frozen=True)
class KsParams:
    """Derived evaluation parameters (ksint.py:48-79)."""

    len_f: int
    len_g: int
    coeff_bits: int
    log2_min_len: int
    width_full: int
    width_half: int
    width_quarter: int

    @property
    def out_len(self) -> int:
        return self.len_f + self.len_g - 1

    @property
    def out_bound_bits(self) -> int:
        return self.width_full

    def coeff_product_bound(self) -> int:
        top = (1 << self.coeff_bits) - 1
        return min(self.len_f, self.len_g) * top * top


@dataclass(frozen=True)
class OverlapDigits:
    """Digit streams feeding the overlap reconstruction (ksint.py:101-134)."""

    forward_digits: tuple
    reversed_digits: tuple
    width_bits: int

    def __post_init__(self):
        object.__setattr__(self, "forward_digits", tuple(int(d) for d in self.forward_digits))
        object.__setattr__(self, "reversed_digits", tuple(int(d) for d in self.reversed_digits))
        if self.width_bits < 1:
            raise ValueError("digit width must be >= 1")
        if len(self.forward_digits) != len(self.reversed_digits):
            raise ValueError("digit streams must have equal length")
        if len(self.forward_digits) < 2:
            raise ValueError("need at least two digits per stream")
        top = 1 << self.width_bits
        for d in self.forward_digits + self.reversed_digits:
            if not 0 <= d < top:
                raise ValueError("digit out of range")

    @property
    def coeff_count(self) -> int:
        return len(self.forward_digits) - 1
