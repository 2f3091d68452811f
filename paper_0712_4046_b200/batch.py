"""Batched API over device tensors (the benchmarked interface).

``KsBatch`` multiplies ``batch`` independent polynomial pairs with one KS
variant in one stream-ordered call: f, g are CUDA int32 tensors holding the
little-endian 32-bit words of each coefficient ([batch, len, in_words]);
the result is [batch, len_f + len_g - 1, out_words].  ``ks_mul_host`` is the
same through host (numpy / pinned) buffers with the copies inside the call.

PyTorch only provides device memory and streams here; all compute is in
libkmx.so (include/kmx.h).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import KMX_SIGNED, check, lib

VARIANTS = {1: "ks1 (standard, 2^N)", 2: "ks2 (reciprocal, 2^N and 2^-N)",
            3: "ks3 (negated, +-2^N)", 4: "ks4 (four-point, +-2^N and +-2^-N)"}


def _torch():
    import torch
    return torch


class KsBatch:
    """Plan + workspace for repeated batched KS products of one shape."""

    def __init__(self, variant: int, batch: int, len_f: int, len_g: int, coeff_bits: int,
                 signed: bool = False, device=None, tune: bool = True):
        torch = _torch()
        self.variant, self.batch, self.len_f, self.len_g = variant, batch, len_f, len_g
        self.coeff_bits = coeff_bits
        self.flags = (KMX_SIGNED if signed else 0) | (0 if tune else _lib.KMX_NO_TUNE)
        self.in_words = 1 if signed else (coeff_bits + 31) // 32
        self.out_len = len_f + len_g - 1
        ow = lib().kmx_ks_out_words(len_f, len_g, coeff_bits, self.flags)
        if ow < 0:
            check(ow, "KsBatch")
        self.out_words = ow
        self.ws_bytes = lib().kmx_ks_workspace_bytes(variant, batch, len_f, len_g, coeff_bits, self.flags)
        if self.ws_bytes == 0 and batch > 0:
            raise ValueError("invalid KS problem shape")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.workspace = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=self.device)
        p = (ctypes.c_int64 * 8)()
        check(lib().kmx_ks_params(variant, len_f, len_g, coeff_bits, self.flags, p), "KsBatch")
        self.params = [int(x) for x in p]

    def empty_out(self):
        torch = _torch()
        return torch.empty((self.batch, self.out_len, self.out_words), dtype=torch.int32, device=self.device)

    def __call__(self, f, g, out=None, stream=None):
        torch = _torch()
        assert f.is_cuda and g.is_cuda and f.dtype == torch.int32 and g.dtype == torch.int32
        assert f.is_contiguous() and g.is_contiguous()
        assert tuple(f.shape) == (self.batch, self.len_f, self.in_words), f.shape
        assert tuple(g.shape) == (self.batch, self.len_g, self.in_words), g.shape
        if out is None:
            out = self.empty_out()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = lib().kmx_ks_mul(self.variant, self.batch, self.len_f, self.len_g, self.coeff_bits,
                              f.data_ptr(), g.data_ptr(), self.in_words, out.data_ptr(), self.out_words,
                              self.workspace.data_ptr(), self.ws_bytes, self.flags, st.cuda_stream)
        check(rc, "kmx_ks_mul")
        return out

    def capture(self, f, g, out=None):
        """Capture this product (fixed buffers) into a CUDA graph; returns
        (graph, out).  ``graph.replay()`` re-runs pack -> multiply -> finish
        [-> reconstruct] with no per-kernel launch overhead."""
        torch = _torch()
        if out is None:
            out = self.empty_out()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self(f, g, out, stream=s)  # warm (attributes, occupancy queries)
        s.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            self(f, g, out, stream=s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return graph, out

    def status(self, stream=None):
        """Synchronise and raise the latched device error, if any."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().kmx_ws_status(self.workspace.data_ptr(), st.cuda_stream), "kmx_ks_mul")

    def limb_products(self, stream=None) -> int:
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        v = ctypes.c_uint64(0)
        check(lib().kmx_ws_limb_products(self.workspace.data_ptr(), self.variant, self.batch, self.len_f,
                                         self.len_g, self.coeff_bits, self.flags, ctypes.byref(v),
                                         st.cuda_stream), "limb_products")
        return int(v.value)


def ks_mul_host(variant: int, f: np.ndarray, g: np.ndarray, coeff_bits: int, signed: bool = False,
                out: np.ndarray | None = None, tune: bool = True) -> np.ndarray:
    """Host-buffer batched KS product: f [batch, len_f, in_words] uint32/int32,
    g [batch, len_g, in_words] -> [batch, len_f+len_g-1, out_words] uint32.
    ``tune=False`` skips the first-call plan measurement (KMX_NO_TUNE)."""
    assert f.ndim == 3 and g.ndim == 3 and f.shape[0] == g.shape[0] and f.shape[2] == g.shape[2]
    batch, lf, iw = f.shape
    lg = g.shape[1]
    flags = (KMX_SIGNED if signed else 0) | (0 if tune else _lib.KMX_NO_TUNE)
    ow = lib().kmx_ks_out_words(lf, lg, coeff_bits, flags)
    if ow < 0:
        check(ow, "ks_mul_host")
    if out is None:
        out = np.empty((batch, lf + lg - 1, ow), dtype=np.uint32)
    assert out.flags.c_contiguous and f.flags.c_contiguous and g.flags.c_contiguous
    rc = lib().kmx_ks_mul_host(variant, batch, lf, lg, coeff_bits, _lib.ptr(f), _lib.ptr(g), iw,
                               _lib.ptr(out), out.shape[2], flags, None)
    check(rc, "kmx_ks_mul_host")
    return out


class BksBatch:
    """Batched bivariate reduction over Z on device tensors: f, g int32
    [batch, lx, ly] -> h int64 [batch, 2lx-1, 2ly-1]."""

    def __init__(self, variant: int, batch: int, lx: int, ly: int, coeff_bits: int, device=None):
        torch = _torch()
        self.variant, self.batch, self.lx, self.ly, self.coeff_bits = variant, batch, lx, ly, coeff_bits
        self.ws_bytes = lib().kmx_bks_workspace_bytes_cb(variant, batch, lx, ly, coeff_bits)
        if self.ws_bytes == 0:
            raise ValueError("invalid bivariate problem shape")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)

    def __call__(self, f, g, out=None, stream=None):
        torch = _torch()
        if out is None:
            out = torch.empty((self.batch, 2 * self.lx - 1, 2 * self.ly - 1), dtype=torch.int64, device=self.device)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = lib().kmx_bks_mul(self.variant, self.batch, self.lx, self.ly, self.coeff_bits, f.data_ptr(),
                               g.data_ptr(), out.data_ptr(), self.workspace.data_ptr(), self.ws_bytes,
                               st.cuda_stream)
        check(rc, "kmx_bks_mul")
        return out

    def capture(self, f, g, out=None):
        """CUDA-graph capture of this bivariate product (see KsBatch.capture)."""
        torch = _torch()
        if out is None:
            out = torch.empty((self.batch, 2 * self.lx - 1, 2 * self.ly - 1), dtype=torch.int64, device=self.device)
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self(f, g, out, stream=s)
        s.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            self(f, g, out, stream=s)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return graph, out

    def status(self, stream=None):
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().kmx_ws_status(self.workspace.data_ptr(), st.cuda_stream), "kmx_bks_mul")


def bks_mul_host(variant: int, f: np.ndarray, g: np.ndarray, coeff_bits: int, out=None) -> np.ndarray:
    batch, lx, ly = f.shape
    if out is None:
        out = np.empty((batch, 2 * lx - 1, 2 * ly - 1), dtype=np.int64)
    rc = lib().kmx_bks_mul_host(variant, batch, lx, ly, coeff_bits, _lib.ptr(f), _lib.ptr(g), _lib.ptr(out))
    check(rc, "kmx_bks_mul_host")
    return out


class BksModBatch:
    """Batched bivariate reduction over Z/nZ on device tensors: f, g int64
    [batch, lx, ly] holding u64 residues in [0, n) -> h [batch, 2lx-1, 2ly-1]
    (u64 residues in int64 storage).  Variants 3 and 4 need odd n."""

    def __init__(self, variant: int, batch: int, lx: int, ly: int, modulus: int, device=None):
        torch = _torch()
        self.variant, self.batch, self.lx, self.ly, self.modulus = variant, batch, lx, ly, modulus
        self.ws_bytes = lib().kmx_bks_mod_workspace_bytes(variant, batch, lx, ly, modulus)
        if self.ws_bytes == 0:
            raise ValueError("invalid bivariate Z/nZ problem (shape, modulus, or even n for variants 3/4)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)

    def __call__(self, f, g, out=None, stream=None):
        torch = _torch()
        assert f.dtype == torch.int64 and g.dtype == torch.int64 and f.is_contiguous() and g.is_contiguous()
        if out is None:
            out = torch.empty((self.batch, 2 * self.lx - 1, 2 * self.ly - 1), dtype=torch.int64, device=self.device)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = lib().kmx_bks_mod_mul(self.variant, self.batch, self.lx, self.ly, self.modulus, f.data_ptr(),
                                   g.data_ptr(), out.data_ptr(), self.workspace.data_ptr(), self.ws_bytes,
                                   st.cuda_stream)
        check(rc, "kmx_bks_mod_mul")
        return out

    def status(self, stream=None):
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().kmx_ws_status(self.workspace.data_ptr(), st.cuda_stream), "kmx_bks_mod_mul")


def imad_peak(iters: int = 4096) -> float:
    """Measured IMAD.WIDE.U32 products/s on the current device."""
    return float(lib().kmx_imad_peak(iters))


def tc_peak(iters: int = 2000) -> float:
    """Measured dense tcgen05 u8 MMA multiply-accumulates/s on the current device."""
    return float(lib().kmx_tc_peak(iters))


def mul_engine(variant: int, len_f: int, len_g: int, coeff_bits: int, signed: bool = False) -> str:
    """Which multiply engine (K2) a product shape runs on: "tensor" or "imad"."""
    rc = lib().kmx_mul_engine(variant, len_f, len_g, coeff_bits, KMX_SIGNED if signed else 0)
    if rc < 0:
        check(rc, "mul_engine")
    return "tensor" if rc == 1 else "imad"


def last_launch_count() -> int:
    return int(lib().kmx_last_launch_count())
