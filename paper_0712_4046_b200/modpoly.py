"""Drop-in (Z/nZ)[x] multiplication on the GPU (kronmul.modpoly).

Mirrors pkg/src/kronmul/modpoly.py: the same ModPoly / Variant /
AutoThresholds / choose_variant / mod_mul names, signatures, validation and
exceptions.  The lift, the KS product and the reduction ``c % n``
(modpoly.py:103-115) all run in libkmx.so (kmx_mod_mul: pack -> multiply ->
finish [-> reconstruct] -> K9 modular reduction); there is no CPU fallback.

``DEFAULT_THRESHOLDS`` keep the reference's bands (48 / 512, modpoly.py:74-75)
so AUTO resolves to the same variant as the reference does.  Results never
depend on the variant.  ``GPU_THRESHOLDS`` are the bands calibrated on B200
from the config-5 crossover sweep (profiles/r01/c5_sweep_final6.json,
tools/calibrate_auto.py).

``ModMulBatch`` / ``mod_mul_host`` are the batched device / host-buffer forms.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from .kstypes import MulConfig, MulStats

__all__ = ["ModPoly", "Variant", "AutoThresholds", "DEFAULT_THRESHOLDS", "GPU_THRESHOLDS",
           "mod_mul", "choose_variant", "ModMulBatch", "mod_mul_host"]

_WORD_BITS = 64


class Variant(enum.Enum):
    KS1 = "ks1"
    KS2 = "ks2"
    KS3 = "ks3"
    KS4 = "ks4"
    AUTO = "auto"


_VARIANT_NUM = {Variant.KS1: 1, Variant.KS2: 2, Variant.KS3: 3, Variant.KS4: 4}


@dataclass(frozen=True)
class ModPoly:
    """Dense polynomial over Z/nZ, constant term first, n in one machine word
    (modpoly.py:41-61)."""

    coeffs: tuple
    modulus: int

    def __post_init__(self):
        coeffs = tuple(int(c) for c in self.coeffs)
        object.__setattr__(self, "coeffs", coeffs)
        n = self.modulus
        if n < 2:
            raise ValueError("modulus must be >= 2")
        if n.bit_length() > _WORD_BITS:
            raise ValueError(f"modulus must fit in {_WORD_BITS} bits")
        if len(coeffs) < 1:
            raise ValueError("a polynomial has length >= 1")
        for i, c in enumerate(coeffs):
            if not 0 <= c < n:
                raise ValueError(f"coefficient {i} outside [0, {n})")

    def __len__(self) -> int:
        return len(self.coeffs)


@dataclass(frozen=True)
class AutoThresholds:
    """Length bands for AUTO variant selection (modpoly.py:64-76): ks1 up to
    ``ks1_max_length``, ks3 up to ``ks3_max_length``, ks4 beyond."""

    ks1_max_length: int = 48
    ks3_max_length: int = 512


DEFAULT_THRESHOLDS = AutoThresholds()
# B200 bands from the config-5 sweep (tools/calibrate_auto.py over
# profiles/r01/c5_sweep_final6.json, coefficient widths 8..64 bits): the band
# edges that minimise the time lost against the per-point fastest variant
# (2.1% mean loss).
GPU_THRESHOLDS = AutoThresholds(ks1_max_length=64, ks3_max_length=1024)


def choose_variant(length: int, coeff_bits: int, thresholds: AutoThresholds | None = None) -> Variant:
    """Deterministic band lookup (modpoly.py:79-92)."""
    if length < 1 or coeff_bits < 1:
        raise ValueError("length and coefficient bits must be >= 1")
    t = thresholds or DEFAULT_THRESHOLDS
    if length <= t.ks1_max_length:
        return Variant.KS1
    if length <= t.ks3_max_length:
        return Variant.KS3
    return Variant.KS4


def _coeff_bits(n: int) -> int:
    return max(1, (n - 1).bit_length())


def mod_mul(f: ModPoly, g: ModPoly, variant: Variant = Variant.AUTO, *,
            thresholds: AutoThresholds | None = None, stats: MulStats | None = None,
            config: MulConfig | None = None, parallel: bool = False) -> ModPoly:
    """f * g mod n; the result has length len(f) + len(g) - 1
    (modpoly.py:95-115).  ``config`` and ``parallel`` are accepted for
    signature compatibility; results never depend on them."""
    if f.modulus != g.modulus:
        raise ValueError("modulus mismatch")
    n = f.modulus
    if variant is Variant.AUTO:
        variant = choose_variant(max(len(f), len(g)), _coeff_bits(n), thresholds)
    v = _VARIANT_NUM[variant]
    lf, lg = len(f.coeffs), len(g.coeffs)
    fa = np.array(f.coeffs, dtype=np.uint64)
    ga = np.array(g.coeffs, dtype=np.uint64)
    h = np.zeros(lf + lg - 1, dtype=np.uint64)
    lp = ctypes.c_uint64(0)
    rc = lib().kmx_mod_mul_host(v, 1, lf, lg, n, _lib.ptr(fa), _lib.ptr(ga), _lib.ptr(h),
                                ctypes.byref(lp) if stats is not None else None)
    check(rc, "mod_mul")
    if stats is not None:
        stats.limb_products += int(lp.value)
    return ModPoly(tuple(int(x) for x in h), n)


def _torch():
    import torch
    return torch


class ModMulBatch:
    """Batched (Z/nZ)[x] products on device tensors: f [batch, len_f],
    g [batch, len_g] int64 holding u64 residues in [0, n) -> h
    [batch, len_f + len_g - 1] (u64 residues in int64 storage)."""

    def __init__(self, variant, batch: int, len_f: int, len_g: int, modulus: int, device=None):
        torch = _torch()
        if isinstance(variant, Variant):
            if variant is Variant.AUTO:
                variant = choose_variant(max(len_f, len_g), _coeff_bits(modulus), GPU_THRESHOLDS)
            variant = _VARIANT_NUM[variant]
        if modulus < 2 or modulus.bit_length() > _WORD_BITS:
            raise ValueError("modulus must satisfy 2 <= n < 2**64")
        self.variant, self.batch, self.len_f, self.len_g, self.modulus = variant, batch, len_f, len_g, modulus
        self.ws_bytes = lib().kmx_mod_workspace_bytes(variant, batch, len_f, len_g, modulus)
        if self.ws_bytes == 0:
            raise ValueError("invalid (Z/nZ)[x] problem shape")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)

    def empty_out(self):
        torch = _torch()
        return torch.empty((self.batch, self.len_f + self.len_g - 1), dtype=torch.int64, device=self.device)

    def __call__(self, f, g, out=None, stream=None):
        torch = _torch()
        assert f.is_cuda and g.is_cuda and f.dtype == torch.int64 and g.dtype == torch.int64
        assert f.is_contiguous() and g.is_contiguous()
        assert tuple(f.shape) == (self.batch, self.len_f) and tuple(g.shape) == (self.batch, self.len_g)
        if out is None:
            out = self.empty_out()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = lib().kmx_mod_mul(self.variant, self.batch, self.len_f, self.len_g, self.modulus, f.data_ptr(),
                               g.data_ptr(), out.data_ptr(), self.workspace.data_ptr(), self.ws_bytes,
                               st.cuda_stream)
        check(rc, "kmx_mod_mul")
        return out

    def status(self, stream=None):
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().kmx_ws_status(self.workspace.data_ptr(), st.cuda_stream), "kmx_mod_mul")


def mod_mul_host(variant: int, f: np.ndarray, g: np.ndarray, modulus: int, out: np.ndarray | None = None) -> np.ndarray:
    """Host-buffer batched (Z/nZ)[x] product: f [batch, len_f], g [batch, len_g]
    uint64 -> [batch, len_f + len_g - 1] uint64."""
    assert f.ndim == 2 and g.ndim == 2 and f.shape[0] == g.shape[0]
    f = np.ascontiguousarray(f, dtype=np.uint64)
    g = np.ascontiguousarray(g, dtype=np.uint64)
    batch, lf = f.shape
    lg = g.shape[1]
    if out is None:
        out = np.empty((batch, lf + lg - 1), dtype=np.uint64)
    rc = lib().kmx_mod_mul_host(variant, batch, lf, lg, modulus, _lib.ptr(f), _lib.ptr(g), _lib.ptr(out), None)
    check(rc, "kmx_mod_mul_host")
    return out
