"""CPU oracle for the multipoint Kronecker-substitution hot path.

TEST INFRASTRUCTURE ONLY.  This module is a checker: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` leg may import it.  The product path (``paper_0712_4046_b200``)
never imports, calls or links anything under ``oracle/``.

It restates, in plain Python integers (the reference's own arithmetic
substrate, ``bignat.py:4-8``), the algorithm of the reference package
``kronmul`` (``/root/reference/pkg/src/kronmul``), function by function.
Each function cites the reference ``file:line`` it follows.  No reference
source is imported or copied; parity of this restatement with the reference is
pinned by ``tests/test_oracle_golden.py`` against the reference's own
known-answer tests and against fixtures generated from the reference itself
(``tests/golden/make_golden.py``).

Two multiply back ends are offered:

* ``mul_mode="karatsuba"`` (default) restates ``bignat._mul_int`` /
  ``_karatsuba_int`` / ``_classical_int`` (``bignat.py:323-371``): 64-bit limb
  schoolbook rows below a 16-limb threshold, additive Karatsuba above.  This
  is what the CPU baseline times, so the baseline has the reference's cost
  structure.
* ``mul_mode="native"`` uses CPython's ``int.__mul__`` directly (the same
  exact product; faster for the large parity checks).
"""

from __future__ import annotations

import operator
from dataclasses import dataclass

LIMB64 = 64
_LIMB64_MASK = (1 << LIMB64) - 1


class OracleReconstructionError(ArithmeticError):
    """Mirrors ``ksint.ReconstructionError`` (``ksint.py:44-45``)."""


class OracleMissingHalve(ValueError):
    """Mirrors ``bipoly.MissingHalveError`` (``bipoly.py:26-28``)."""


# --------------------------------------------------------------------------
# parameters  (ksint.py:48-98, :214-216, :282-286)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Params:
    len_f: int
    len_g: int
    b: int
    e: int
    n1: int   # width_full  = 2b+e
    n2: int   # width_half  = b + ceil(e/2)
    n4: int   # width_quarter = ceil((2b+e)/4)

    @property
    def out_len(self) -> int:
        return self.len_f + self.len_g - 1


def derive_params(len_f: int, len_g: int, b: int) -> Params:
    """ksint.py:82-98."""
    if len_f < 1 or len_g < 1:
        raise ValueError("polynomial lengths must be >= 1")
    if b < 1:
        raise ValueError("coefficient bit bound must be >= 1")
    e = (min(len_f, len_g) - 1).bit_length()
    n1 = 2 * b + e
    return Params(len_f, len_g, b, e, n1, b + (e + 1) // 2, (n1 + 3) // 4)


def four_point_safe(p: Params) -> bool:
    """ksint.py:282-286: min(L)(2^b-1)^2 < 2^w (2^w - 1), w = 2 N4."""
    w = 2 * p.n4
    top = (1 << p.b) - 1
    return min(p.len_f, p.len_g) * top * top < (1 << w) * ((1 << w) - 1)


# --------------------------------------------------------------------------
# digit blits  (bignat.py:411-450)
# --------------------------------------------------------------------------

def pack_ints(values, width: int) -> int:
    """sum(v_i 2^(i width)), built from groups of 8 digits (8*width bits =
    width bytes) joined as bytes -- linear time, bignat.py:411-428."""
    if width < 1:
        raise ValueError("digit width must be >= 1")
    values = list(values)
    if not values:
        return 0
    parts = []
    for start in range(0, len(values), 8):
        group = 0
        for j, v in enumerate(values[start:start + 8]):
            group |= v << (j * width)
        parts.append(group.to_bytes(width, "little"))
    return int.from_bytes(b"".join(parts), "little")


def unpack_ints(value: int, width: int, count: int) -> list[int]:
    """Base-2^width digits, least significant first; raises if the value
    does not fit in ``count`` digits (bignat.py:431-450)."""
    if width < 1 or count < 0:
        raise ValueError("bad digit width/count")
    if value < 0 or value.bit_length() > width * count:
        raise ValueError(f"value does not fit in {count} digits of {width} bits")
    if count == 0:
        return []
    ngroups = (count + 7) // 8
    raw = value.to_bytes(ngroups * width, "little")
    mask = (1 << width) - 1
    out = []
    for g in range(ngroups):
        acc = int.from_bytes(raw[g * width:(g + 1) * width], "little")
        for _ in range(8):
            out.append(acc & mask)
            acc >>= width
    return out[:count]


# --------------------------------------------------------------------------
# evaluation packing  (pack.py:55-110)
# --------------------------------------------------------------------------

def _check_width(b: int, width: int) -> None:
    """pack.py:55-59."""
    if 2 * width < b:
        raise ValueError(f"chunk width {width} below half the coefficient bound {b}")


def value_at_pow2(coeffs, width: int, b: int) -> int:
    """pack.py:62-69: single blit if width >= b, else even + (odd << width)."""
    if width >= b:
        return pack_ints(coeffs, width)
    return pack_ints(coeffs[0::2], 2 * width) + (pack_ints(coeffs[1::2], 2 * width) << width)


def value_at_neg_pow2(coeffs, width: int) -> int:
    """pack.py:72-76: even - (odd << width), signed."""
    return pack_ints(coeffs[0::2], 2 * width) - (pack_ints(coeffs[1::2], 2 * width) << width)


def pack(coeffs, width: int, b: int) -> int:
    """pack.py:79-82 (value at 2^N)."""
    _check_width(b, width)
    return value_at_pow2(list(coeffs), width, b)


def pack_reversed(coeffs, width: int, b: int) -> int:
    """pack.py:85-90 (value at 2^-N, normalized)."""
    _check_width(b, width)
    return value_at_pow2(list(coeffs)[::-1], width, b)


def pack_negated(coeffs, width: int, b: int) -> int:
    """pack.py:93-96 (value at -2^N, signed)."""
    _check_width(b, width)
    return value_at_neg_pow2(list(coeffs), width)


def pack_negated_reversed(coeffs, width: int, b: int) -> int:
    """pack.py:99-110 (value at -2^-N, normalized; sign flip for even L)."""
    _check_width(b, width)
    v = value_at_neg_pow2(list(coeffs)[::-1], width)
    return -v if len(coeffs) % 2 == 0 else v


# --------------------------------------------------------------------------
# multiplication  (bignat.py:323-380, :397-401)
# --------------------------------------------------------------------------

class Counter:
    """Mirrors ``MulStats.limb_products`` (bignat.py:57-68): 64-bit word
    products performed."""

    def __init__(self):
        self.limb_products = 0


def _nlimbs64(x: int) -> int:
    return (x.bit_length() + LIMB64 - 1) // LIMB64


def mul_classical(x: int, y: int, stats: Counter | None = None) -> int:
    """bignat.py:323-341: one shifted row per 64-bit limb of the shorter
    operand; counts limbs(x)*limbs(y)."""
    xl, yl = _nlimbs64(x), _nlimbs64(y)
    if stats is not None:
        stats.limb_products += xl * yl
    if xl == 0 or yl == 0:
        return 0
    if xl > yl:
        x, y, xl = y, x, yl
    acc = 0
    for i in range(xl):
        w = (x >> (i * LIMB64)) & _LIMB64_MASK
        if w:
            acc += (w * y) << (i * LIMB64)
    return acc


def mul_karatsuba(x: int, y: int, stats: Counter | None, threshold: int = 16) -> int:
    """bignat.py:344-363: split at half the longer operand (rounded up),
    z1 = (x0+x1)(y0+y1) - z0 - z2."""
    xl, yl = _nlimbs64(x), _nlimbs64(y)
    if xl <= threshold or yl <= threshold:
        return mul_classical(x, y, stats)
    half = (max(xl, yl) + 1) // 2
    s = half * LIMB64
    m = (1 << s) - 1
    x0, x1, y0, y1 = x & m, x >> s, y & m, y >> s
    z0 = mul_karatsuba(x0, y0, stats, threshold)
    z2 = mul_karatsuba(x1, y1, stats, threshold)
    z1 = mul_karatsuba(x0 + x1, y0 + y1, stats, threshold) - z0 - z2
    return z0 + (z1 << s) + (z2 << (2 * s))


def mul(x: int, y: int, mode: str = "karatsuba", stats: Counter | None = None,
        threshold: int = 16, classical_only: bool = False) -> int:
    """bignat.py:366-380 dispatch (magnitudes; sign handled by the caller as
    in mul_signed, bignat.py:397-401)."""
    sign = (x < 0) ^ (y < 0)
    ax, ay = abs(x), abs(y)
    if mode == "native":
        r = ax * ay
    elif classical_only or min(_nlimbs64(ax), _nlimbs64(ay)) <= threshold:
        r = mul_classical(ax, ay, stats)
    else:
        r = mul_karatsuba(ax, ay, stats, threshold)
    return -r if sign else r


# --------------------------------------------------------------------------
# exact halving / shifting  (bignat.py:265-274, :310-317)
# --------------------------------------------------------------------------

def halve_exact(v: int) -> int:
    """SignedBig.halve_exact + to_bignat (bignat.py:265-274)."""
    if v & 1:
        raise ValueError("halving an odd value is not exact")
    v >>= 1
    if v < 0:
        raise ValueError("negative value cannot become a BigNat")
    return v


def shr_exact(v: int, k: int) -> int:
    """bignat.py:310-317."""
    if v & ((1 << k) - 1):
        raise ValueError(f"inexact shift: low {k} bits are not all zero")
    return v >> k


# --------------------------------------------------------------------------
# overlap reconstruction  (ksint.py:137-179)
# --------------------------------------------------------------------------

def reconstruct(fwd, rev, width: int):
    """The alpha/beta/delta/epsilon solve of ksint.py:137-179.

    ``fwd``: base-2^width digits of sum h_i 2^(i w), least significant first;
    ``rev``: digits of the reversed sum listed most significant first.
    Returns (coeffs, forward_carries, reverse_carries)."""
    count = len(fwd) - 1
    base = 1 << width
    mask = base - 1
    lo = [0] * count
    hi = [0] * count
    fc = [0] * (count + 1)
    rc = [0] * count
    lo[0] = fwd[0]
    for j in range(count - 1):
        eps = 1 if lo[j] > rev[j + 1] else 0           # ksint.py:154 (strict)
        rc[j] = eps
        h = (rev[j] - (lo[j - 1] if j else 0) - eps) & mask
        if h >= mask:
            raise OracleReconstructionError("high digit out of range")
        hi[j] = h
        nxt = (fwd[j + 1] - h - fc[j]) & mask
        lo[j + 1] = nxt
        t = h + nxt + fc[j] - fwd[j + 1]
        if t == 0:
            fc[j + 1] = 0
        elif t == base:
            fc[j + 1] = 1
        else:
            raise OracleReconstructionError("forward carry out of range")
    h = (rev[count - 1] - (lo[count - 2] if count >= 2 else 0)) & mask
    if h >= mask:
        raise OracleReconstructionError("high digit out of range")
    hi[count - 1] = h
    if lo[count - 1] != rev[count]:
        raise OracleReconstructionError("digit streams disagree")
    if h + fc[count - 1] != fwd[count]:
        raise OracleReconstructionError("top digit mismatch")
    return [lo[i] | (hi[i] << width) for i in range(count)], fc, rc


def _interleave(even, odd):
    """ksint.py:250-254."""
    out = [0] * (len(even) + len(odd))
    out[0::2] = even
    out[1::2] = odd
    return out


# --------------------------------------------------------------------------
# the four integer variants  (ksint.py:219-348)
# --------------------------------------------------------------------------

def ks1(f, g, b: int, mode: str = "karatsuba", stats: Counter | None = None,
        classical_only: bool = False) -> list[int]:
    """ksint.py:219-226: pack at N1, one product, unpack out_len digits."""
    p = derive_params(len(f), len(g), b)
    n = p.n1
    prod = mul(pack(f, n, b), pack(g, n, b), mode, stats, classical_only=classical_only)
    return unpack_ints(prod, n, p.out_len)


def ks2(f, g, b: int, mode: str = "karatsuba", stats: Counter | None = None,
        classical_only: bool = False) -> list[int]:
    """ksint.py:229-247 (reciprocal): forward and reversed products at N2,
    out_len+1 digits each, reversed list flipped, reconstruction."""
    p = derive_params(len(f), len(g), b)
    n = p.n2
    pf = mul(pack(f, n, b), pack(g, n, b), mode, stats, classical_only=classical_only)
    pr = mul(pack_reversed(f, n, b), pack_reversed(g, n, b), mode, stats,
             classical_only=classical_only)
    nd = p.out_len + 1
    fwd = unpack_ints(pf, n, nd)
    rev = unpack_ints(pr, n, nd)[::-1]
    return reconstruct(fwd, rev, n)[0]


def ks3(f, g, b: int, mode: str = "karatsuba", stats: Counter | None = None,
        classical_only: bool = False) -> list[int]:
    """ksint.py:257-279 (negated): products at +-2^N2; half-sum holds the
    even coefficients, half-difference >> N2 the odd ones."""
    p = derive_params(len(f), len(g), b)
    n = p.n2
    pos = mul(pack(f, n, b), pack(g, n, b), mode, stats, classical_only=classical_only)
    neg = mul(pack_negated(f, n, b), pack_negated(g, n, b), mode, stats,
              classical_only=classical_only)
    even_v = halve_exact(pos + neg)
    odd_v = shr_exact(halve_exact(pos - neg), n)
    k = p.out_len
    even = unpack_ints(even_v, 2 * n, (k + 1) // 2)
    odd = unpack_ints(odd_v, 2 * n, k // 2)
    return _interleave(even, odd)


def ks4(f, g, b: int, mode: str = "karatsuba", stats: Counter | None = None,
        classical_only: bool = False) -> list[int]:
    """ksint.py:289-348 (four-point): quarter-width products at +-2^N4 and
    +-2^-N4, even/odd split, two reconstructions at width 2 N4.  Falls back
    to ks1 when the bound is not certified (ksint.py:299-300); out_len == 1
    is a single product (ksint.py:301-303)."""
    p = derive_params(len(f), len(g), b)
    if not four_point_safe(p):
        return ks1(f, g, b, mode, stats, classical_only)
    if p.out_len == 1:
        return [mul(f[0], g[0], mode, stats, classical_only=classical_only)]
    n = p.n4
    w = 2 * n
    pf = mul(pack(f, n, b), pack(g, n, b), mode, stats, classical_only=classical_only)
    pn = mul(pack_negated(f, n, b), pack_negated(g, n, b), mode, stats,
             classical_only=classical_only)
    pr = mul(pack_reversed(f, n, b), pack_reversed(g, n, b), mode, stats,
             classical_only=classical_only)
    pnr = mul(pack_negated_reversed(f, n, b), pack_negated_reversed(g, n, b), mode,
              stats, classical_only=classical_only)
    k = p.out_len
    n_even, n_odd = (k + 1) // 2, k // 2
    fwd_even = halve_exact(pf + pn)
    fwd_odd = shr_exact(halve_exact(pf - pn), n)
    rev_even = halve_exact(pr + pnr)
    rev_odd = halve_exact(pr - pnr)
    if k % 2 == 0:                                  # ksint.py:332-335
        rev_even = shr_exact(rev_even, n)
    else:
        rev_odd = shr_exact(rev_odd, n)
    even = reconstruct(unpack_ints(fwd_even, w, n_even + 1),
                       unpack_ints(rev_even, w, n_even + 1)[::-1], w)[0]
    if n_odd:
        odd = reconstruct(unpack_ints(fwd_odd, w, n_odd + 1),
                          unpack_ints(rev_odd, w, n_odd + 1)[::-1], w)[0]
    else:
        odd = []
    return _interleave(even, odd)


KS = {1: ks1, 2: ks2, 3: ks3, 4: ks4}


def ks_mul(variant: int, f, g, b: int, mode: str = "karatsuba", stats=None,
           classical_only: bool = False) -> list[int]:
    return KS[variant](list(f), list(g), b, mode, stats, classical_only)


# --------------------------------------------------------------------------
# signed inputs: bias lift through the unsigned variants
# --------------------------------------------------------------------------

def ks_mul_signed(variant: int, f, g, b: int, mode: str = "karatsuba") -> list[int]:
    """Signed b-bit coefficients (two's complement range [-2^(b-1), 2^(b-1))).
    The reference rejects negative coefficients (pack.py:44-46), so the
    signed product is obtained from the reference's unsigned variant on the
    lifted inputs f' = f + B, g' = g + B (B = 2^(b-1), bound b):
    h = h' - B (J*f' + J*g') + B^2 (J*J), J the all-ones vector."""
    bias = 1 << (b - 1)
    fl = [c + bias for c in f]
    gl = [c + bias for c in g]
    h = ks_mul(variant, fl, gl, b, mode)
    lf, lg = len(f), len(g)
    # sliding-window sums: (J_lg * f')_k = sum_{i: 0 <= k-i < lg} f'_i
    pf = [0]
    for c in fl:
        pf.append(pf[-1] + c)
    pg = [0]
    for c in gl:
        pg.append(pg[-1] + c)
    out = []
    for k in range(lf + lg - 1):
        sf = pf[min(k, lf - 1) + 1] - pf[max(0, k - lg + 1)]
        sg = pg[min(k, lg - 1) + 1] - pg[max(0, k - lf + 1)]
        cnt = min(k, lf - 1) - max(0, k - lg + 1) + 1
        out.append(h[k] - bias * (sf + sg) + bias * bias * cnt)
    return out


# --------------------------------------------------------------------------
# (Z/nZ)[x]  (modpoly.py:79-115, oracle.py:30-40)
# --------------------------------------------------------------------------

def mod_coeff_bits(n: int) -> int:
    """modpoly.py:104: the lift's bound comes from the modulus, not the data."""
    return max(1, (n - 1).bit_length())


def choose_variant(length: int, coeff_bits: int, ks1_max: int = 48, ks3_max: int = 512) -> int:
    """modpoly.py:79-92 (band lookup; defaults modpoly.py:74-75)."""
    if length < 1 or coeff_bits < 1:
        raise ValueError("length and coefficient bits must be >= 1")
    if length <= ks1_max:
        return 1
    if length <= ks3_max:
        return 3
    return 4


def mod_mul(variant: int, f, g, n: int, mode: str = "karatsuba", stats=None,
            classical_only: bool = False) -> list[int]:
    """modpoly.py:95-115: lift to Z with b = bitlen(n-1), KS product, reduce
    every coefficient mod n.  variant 0 = AUTO (reference thresholds)."""
    if n < 2:
        raise ValueError("modulus must be >= 2")
    for c in list(f) + list(g):
        if not 0 <= c < n:
            raise ValueError("coefficient outside [0, n)")
    b = mod_coeff_bits(n)
    if variant == 0:
        variant = choose_variant(max(len(f), len(g)), b)
    return [c % n for c in ks_mul(variant, f, g, b, mode, stats, classical_only)]


def schoolbook_mod(f, g, n: int) -> list[int]:
    """oracle.py:30-40: word-modular convolution."""
    out = [0] * (len(f) + len(g) - 1)
    for i, a in enumerate(f):
        if a:
            for j, c in enumerate(g):
                out[i + j] = (out[i + j] + a * c) % n
    return out


# --------------------------------------------------------------------------
# brute-force convolution  (oracle.py:19-27, :58-69)
# --------------------------------------------------------------------------

def schoolbook(f, g) -> list[int]:
    """oracle.py:19-27: h[k] = sum_{i+j=k} f[i] g[j] (exact Python ints)."""
    out = [0] * (len(f) + len(g) - 1)
    for i, a in enumerate(f):
        if a:
            for j, c in enumerate(g):
                out[i + j] += a * c
    return out


def uni_schoolbook(a, b) -> list[int]:
    """oracle.py:58-69 with ring_z(): the reference's default univariate
    multiplier for the bivariate reductions (bipoly.py:121-125), a plain
    double loop through the ring callbacks -- kept with that cost structure
    for the CPU baseline of config 3."""
    add, mul = operator.add, operator.mul
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] = add(out[i + j], mul(x, y))
    return out


def convolve_exact(a, b) -> list[int]:
    """Exact integer convolution for the univariate products of the
    bivariate reductions (the role of ``uni_schoolbook`` over Z,
    oracle.py:58-69).  Uses numpy int64 when the result provably fits,
    else Python ints."""
    import numpy as np
    if not a or not b:
        return []
    ma = max(abs(int(x)) for x in a)
    mb = max(abs(int(x)) for x in b)
    if ma * mb * min(len(a), len(b)) < (1 << 62):
        r = np.convolve(np.asarray(a, dtype=np.int64), np.asarray(b, dtype=np.int64))
        return [int(x) for x in r]
    return schoolbook(a, b)


# --------------------------------------------------------------------------
# bivariate reductions R[x,y] -> R[x] over R = Z  (bipoly.py:100-278)
# --------------------------------------------------------------------------

def _ychunks(c):
    """bipoly.py:100-103: chunk j = x-vector of y^j; c is [lx][ly]."""
    lx, ly = len(c), len(c[0])
    return [[c[i][j] for i in range(lx)] for j in range(ly)]


def _from_ychunks(chunks):
    """bipoly.py:106-108."""
    lx = len(chunks[0])
    return [[chunks[j][i] for j in range(len(chunks))] for i in range(lx)]


def _concat(chunks, spacing, chunk_len, reverse=False, alternate=False):
    """bipoly.py:128-143."""
    count = len(chunks)
    vec = [0] * (spacing * (count - 1) + chunk_len)
    for k, ch in enumerate(chunks):
        base = (count - 1 - k if reverse else k) * spacing
        sgn = -1 if (alternate and k % 2 == 1) else 1
        for t, c in enumerate(ch):
            vec[base + t] += sgn * c
    return vec


def _split(vec, spacing, chunk_len, count):
    """bipoly.py:146-148."""
    return [list(vec[k * spacing:k * spacing + chunk_len]) for k in range(count)]


def _overlap_recover(fwd, rev, count, spacing, chunk_len):
    """bipoly.py:151-174."""
    fwd, rev = list(fwd), list(rev)
    out = []
    low = min(spacing, chunk_len)
    for k in range(count):
        fpos, rpos = k * spacing, (count - 1 - k) * spacing
        chunk = fwd[fpos:fpos + low]
        if chunk_len > spacing:
            chunk += rev[rpos + spacing:rpos + chunk_len]
        for t, c in enumerate(chunk):
            fwd[fpos + t] -= c
            rev[rpos + t] -= c
        out.append(chunk)
    return out


def _halve(v):
    if v & 1:
        raise ValueError("halving an odd integer is not exact")
    return v >> 1


def bks(variant: int, f, g, umul=convolve_exact):
    """bipoly.py:177-278 with ring_z() (bipoly.py:53-56).  variant: 1
    standard, 2 reciprocal, 3 negated, 4 four-point.  f, g: [lx][ly]."""
    lx, ly = len(f), len(f[0])
    if len(g) != lx or len(g[0]) != ly:
        raise ValueError("inputs must share both lengths")
    cf, cg = _ychunks(f), _ychunks(g)
    if variant == 1:                                       # :177-188
        sp = 2 * lx - 1
        prod = umul(_concat(cf, sp, lx), _concat(cg, sp, lx))
        return _from_ychunks(_split(prod, sp, 2 * lx - 1, 2 * ly - 1))
    if variant == 2:                                       # :191-206
        pf = umul(_concat(cf, lx, lx), _concat(cg, lx, lx))
        pr = umul(_concat(cf, lx, lx, reverse=True), _concat(cg, lx, lx, reverse=True))
        return _from_ychunks(_overlap_recover(pf, pr, 2 * ly - 1, lx, 2 * lx - 1))
    if variant == 3:                                       # :209-232
        pp = umul(_concat(cf, lx, lx), _concat(cg, lx, lx))
        pn = umul(_concat(cf, lx, lx, alternate=True), _concat(cg, lx, lx, alternate=True))
        ev = [_halve(a + c) for a, c in zip(pp, pn)]
        od = [_halve(a - c) for a, c in zip(pp, pn)][lx:]
        chunks = [None] * (2 * ly - 1)
        chunks[0::2] = _split(ev, 2 * lx, 2 * lx - 1, ly)
        chunks[1::2] = _split(od, 2 * lx, 2 * lx - 1, ly - 1)
        return _from_ychunks(chunks)
    if variant == 4:                                       # :235-278
        if lx == 1 and ly == 1:
            return [[umul([f[0][0]], [g[0][0]])[0]]]
        n = (lx + 1) // 2

        def points(ch):
            return (_concat(ch, n, lx), _concat(ch, n, lx, alternate=True),
                    _concat(ch, n, lx, reverse=True),
                    _concat(ch, n, lx, reverse=True, alternate=True))
        pa, pb = points(cf), points(cg)
        pp, pn, prp, prn = (umul(x, y) for x, y in zip(pa, pb))
        fe = [_halve(a + c) for a, c in zip(pp, pn)]
        fo = [_halve(a - c) for a, c in zip(pp, pn)][n:]
        re_ = [_halve(a + c) for a, c in zip(prp, prn)]
        ro = [_halve(a - c) for a, c in zip(prp, prn)][n:]
        even = _overlap_recover(fe, re_, ly, 2 * n, 2 * lx - 1)
        odd = _overlap_recover(fo, ro, ly - 1, 2 * n, 2 * lx - 1) if ly > 1 else []
        chunks = [None] * (2 * ly - 1)
        chunks[0::2] = even
        chunks[1::2] = odd
        return _from_ychunks(chunks)
    raise ValueError("variant must be 1..4")


def bks_mod(variant: int, f, g, n: int, umul=None):
    """bipoly.py:177-278 with ring_zmod(n) (bipoly.py:59-72): the same steps
    as ``bks`` in the ring's arithmetic -- additions and subtractions mod n,
    halving a * (n+1)/2 mod n (odd n only; bipoly.py:64-66, MissingHalveError
    :116-118) -- with the reference's default UniMul (uni_schoolbook over the
    ring, oracle.py:58-69) unless ``umul`` is given.  Inputs are ring elements
    (reduced mod n here, as the ring's own ops would)."""
    if n < 2:
        raise ValueError("modulus must be >= 2")
    lx, ly = len(f), len(f[0])
    if len(g) != lx or len(g[0]) != ly:
        raise ValueError("inputs must share both lengths")
    if variant in (3, 4) and n % 2 == 0:
        raise ValueError("MissingHalveError: ring does not support exact halving")
    f = [[c % n for c in row] for row in f]
    g = [[c % n for c in row] for row in g]
    inv2 = (n + 1) // 2

    def hv(a):
        return (a * inv2) % n

    def mul(a, b):
        if umul is not None:
            return [c % n for c in umul(a, b)]
        out = [0] * (len(a) + len(b) - 1)
        for i, x in enumerate(a):
            for j, y in enumerate(b):
                out[i + j] = (out[i + j] + (x * y) % n) % n
        return out

    def cat(chunks, spacing, chunk_len, reverse=False, alternate=False):
        v = _concat(chunks, spacing, chunk_len, reverse, alternate)
        return [c % n for c in v]

    def recover(fwd, rev, count, spacing, chunk_len):
        fwd, rev = list(fwd), list(rev)
        out = []
        low = min(spacing, chunk_len)
        for k in range(count):
            fpos, rpos = k * spacing, (count - 1 - k) * spacing
            chunk = fwd[fpos:fpos + low]
            if chunk_len > spacing:
                chunk += rev[rpos + spacing:rpos + chunk_len]
            for t, c in enumerate(chunk):
                fwd[fpos + t] = (fwd[fpos + t] - c) % n
                rev[rpos + t] = (rev[rpos + t] - c) % n
            out.append(chunk)
        return out

    cf, cg = _ychunks(f), _ychunks(g)
    if variant == 1:
        sp = 2 * lx - 1
        return _from_ychunks(_split(mul(cat(cf, sp, lx), cat(cg, sp, lx)), sp, 2 * lx - 1, 2 * ly - 1))
    if variant == 2:
        pf = mul(cat(cf, lx, lx), cat(cg, lx, lx))
        pr = mul(cat(cf, lx, lx, reverse=True), cat(cg, lx, lx, reverse=True))
        return _from_ychunks(recover(pf, pr, 2 * ly - 1, lx, 2 * lx - 1))
    if variant == 3:
        pp = mul(cat(cf, lx, lx), cat(cg, lx, lx))
        pn = mul(cat(cf, lx, lx, alternate=True), cat(cg, lx, lx, alternate=True))
        ev = [hv((a + c) % n) for a, c in zip(pp, pn)]
        od = [hv((a - c) % n) for a, c in zip(pp, pn)][lx:]
        chunks = [None] * (2 * ly - 1)
        chunks[0::2] = _split(ev, 2 * lx, 2 * lx - 1, ly)
        chunks[1::2] = _split(od, 2 * lx, 2 * lx - 1, ly - 1)
        return _from_ychunks(chunks)
    if variant == 4:
        if lx == 1 and ly == 1:
            return [[mul([f[0][0]], [g[0][0]])[0]]]
        h = (lx + 1) // 2

        def points(ch):
            return (cat(ch, h, lx), cat(ch, h, lx, alternate=True),
                    cat(ch, h, lx, reverse=True), cat(ch, h, lx, reverse=True, alternate=True))
        pa, pb = points(cf), points(cg)
        pp, pn, prp, prn = (mul(x, y) for x, y in zip(pa, pb))
        fe = [hv((a + c) % n) for a, c in zip(pp, pn)]
        fo = [hv((a - c) % n) for a, c in zip(pp, pn)][h:]
        re_ = [hv((a + c) % n) for a, c in zip(prp, prn)]
        ro = [hv((a - c) % n) for a, c in zip(prp, prn)][h:]
        even = recover(fe, re_, ly, 2 * h, 2 * lx - 1)
        odd = recover(fo, ro, ly - 1, 2 * h, 2 * lx - 1) if ly > 1 else []
        chunks = [None] * (2 * ly - 1)
        chunks[0::2] = even
        chunks[1::2] = odd
        return _from_ychunks(chunks)
    raise ValueError("variant must be 1..4")


def schoolbook_bivar(f, g):
    """oracle.py:43-55 over Z."""
    lx, ly = len(f), len(f[0])
    out = [[0] * (2 * ly - 1) for _ in range(2 * lx - 1)]
    for i in range(lx):
        for j in range(ly):
            a = f[i][j]
            if a:
                for k in range(lx):
                    for l in range(ly):
                        out[i + k][j + l] += a * g[k][l]
    return out


# --------------------------------------------------------------------------
# limb-array <-> int helpers for batched checks (numpy)
# --------------------------------------------------------------------------

def words_to_ints(arr) -> list:
    """[..., W] little-endian uint32 words -> nested lists of Python ints
    (last axis consumed)."""
    import numpy as np
    a = np.ascontiguousarray(arr, dtype=np.uint32)
    w = a.shape[-1]
    flat = a.reshape(-1, w)
    raw = flat.tobytes()
    step = 4 * w
    vals = [int.from_bytes(raw[i * step:(i + 1) * step], "little") for i in range(flat.shape[0])]
    shape = a.shape[:-1]
    return np.array(vals, dtype=object).reshape(shape).tolist() if shape else vals[0]


def ints_to_words(vals, words: int, signed: bool = False):
    """Nested lists of Python ints -> [..., words] uint32 (two's complement
    when ``signed``)."""
    import numpy as np
    arr = np.array(vals, dtype=object)
    flat = arr.reshape(-1)
    mod = 1 << (32 * words)
    buf = bytearray()
    for v in flat:
        v = int(v)
        if v < 0:
            if not signed:
                raise ValueError("negative value")
            v += mod
        buf += v.to_bytes(4 * words, "little")
    return np.frombuffer(bytes(buf), dtype=np.uint32).reshape(arr.shape + (words,)).copy()
