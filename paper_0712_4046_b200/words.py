"""Conversions between Python integers and little-endian 32-bit word arrays
(the layout of the C ABI: [..., words] uint32)."""
from __future__ import annotations

import numpy as np


def ints_to_words(values, words: int, signed: bool = False) -> np.ndarray:
    """1-D sequence of ints -> [len, words] uint32 (two's complement if signed)."""
    n = len(values)
    nb = 4 * words
    mod = 1 << (32 * words)
    buf = bytearray(n * nb)
    for i, v in enumerate(values):
        v = int(v)
        if v < 0:
            if not signed:
                raise ValueError("negative value in an unsigned word array")
            v += mod
        buf[i * nb:(i + 1) * nb] = v.to_bytes(nb, "little")
    return np.frombuffer(bytes(buf), dtype=np.uint32).reshape(n, words).copy()


def words_to_ints(arr: np.ndarray, signed: bool = False) -> list:
    """[n, words] uint32 -> list of n Python ints."""
    a = np.ascontiguousarray(arr, dtype=np.uint32)
    w = a.shape[-1]
    raw = a.reshape(-1, w).tobytes()
    step = 4 * w
    out = [int.from_bytes(raw[i:i + step], "little") for i in range(0, len(raw), step)]
    if signed:
        top = 1 << (32 * w - 1)
        mod = 1 << (32 * w)
        out = [v - mod if v >= top else v for v in out]
    return out
