"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/kmx.h declares, and its host-only planning functions agree with the
oracle (no device calls)."""
import ctypes
import os
import re

import pytest

from oracle import ks_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_0712_4046_b200 import _lib as L
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("libkmx.so not built (run __graft_entry__.build())")
    return L


def test_header_symbols_exported():
    L = _lib()
    hdr = open(os.path.join(ROOT, "include", "kmx.h")).read()
    declared = set(re.findall(r"\b(kmx_\w+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(L.EXPORTED_SYMBOLS)


def test_params_match_oracle():
    L = _lib()
    out = (ctypes.c_int64 * 8)()
    for lf, lg, b in [(4, 4, 10), (1, 1, 7), (5, 3, 7), (256, 256, 64), (1024, 1024, 32), (4096, 4096, 128),
                      (8192, 8192, 256), (16, 16, 8), (2, 300, 33)]:
        assert L.lib().kmx_ks_params(1, lf, lg, b, 0, out) == 0
        p = O.derive_params(lf, lg, b)
        assert (out[0], out[1], out[2], out[3]) == (p.e, p.n1, p.n2, p.n4)
        assert bool(out[4]) == O.four_point_safe(p)
        assert out[5] == p.out_len


def test_four_point_safe_matches_oracle_grid():
    L = _lib()
    out = (ctypes.c_int64 * 8)()
    for L_ in (1, 2, 3, 5, 16, 64, 255, 256, 257, 1024, 4096, 8192):
        for b in (1, 2, 3, 7, 8, 31, 32, 33, 64, 128, 255, 256):
            assert L.lib().kmx_ks_params(4, L_, L_, b, 0, out) == 0
            assert bool(out[4]) == O.four_point_safe(O.derive_params(L_, L_, b)), (L_, b)


def test_out_words_and_workspace():
    L = _lib()
    assert L.lib().kmx_ks_out_words(256, 256, 64, 0) == 5       # 136 bits
    assert L.lib().kmx_ks_out_words(1024, 1024, 32, 1) == 3     # 74 bits signed
    assert L.lib().kmx_ks_out_words(4096, 4096, 128, 0) == 9    # 268 bits
    for v in (1, 2, 3, 4):
        assert L.lib().kmx_ks_workspace_bytes(v, 64, 256, 256, 64, 0) > 0
    assert L.lib().kmx_ks_workspace_bytes(5, 64, 256, 256, 64, 0) == 0
    assert L.lib().kmx_ks_out_words(0, 4, 4, 0) == L.KMX_EINVAL


def test_error_mapping():
    L = _lib()
    with pytest.raises(ValueError):
        L.check(L.KMX_EINVAL)
    with pytest.raises(ValueError):
        L.check(L.KMX_EINEXACT)
    with pytest.raises(L.ReconstructionError):
        L.check(L.KMX_ERECON)
    with pytest.raises(ArithmeticError):
        L.check(L.KMX_ERECON)
    L.check(L.KMX_OK)


def test_derive_params_dropin():
    _lib()
    import paper_0712_4046_b200 as k
    p = k.derive_params(4, 4, 10)
    assert (p.log2_min_len, p.width_full, p.width_half, p.width_quarter) == (2, 22, 11, 6)
    with pytest.raises(ValueError):
        k.derive_params(0, 1, 4)
    with pytest.raises(ValueError):
        k.derive_params(1, 1, 0)


def test_dropin_types_validate():
    from paper_0712_4046_b200.kstypes import CoeffVec, OverlapDigits
    with pytest.raises(ValueError):
        CoeffVec((), 4)
    with pytest.raises(ValueError):
        CoeffVec((16,), 4)
    with pytest.raises(ValueError):
        CoeffVec((-1,), 4)
    with pytest.raises(ValueError):
        OverlapDigits((1,), (1,), 3)
    with pytest.raises(ValueError):
        OverlapDigits((8, 0), (0, 8), 3)
    assert CoeffVec((0, 15), 4).reversed().coeffs == (15, 0)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_0712_4046_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle.py", ""), fn
