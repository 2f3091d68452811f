"""K1 (the pack kernel) by itself against the reference's own pack values:
tests/golden/pack_golden.json.gz holds pack / pack_reversed / pack_negated /
pack_negated_reversed of 206 vectors computed by kronmul.pack
(pack.py:79-110), including the KATs of pkg/tests/test_pack.py:26-59 and the
overlapped (width < bound) regime.  Plus one batched launch of many vectors
against the oracle restatement, and the width / range errors."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ks_oracle as O  # noqa: E402
from tests import golden_io as G  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kpack():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import importlib
    return importlib.import_module("paper_0712_4046_b200.pack")


def test_pack_golden(kpack):
    from paper_0712_4046_b200.kstypes import CoeffVec
    n = 0
    for coeffs, b, w, pk, rev, neg, nrev in G.pack_cases():
        v = CoeffVec(tuple(coeffs), b)
        assert kpack.pack(v, w) == pk, (coeffs, b, w)
        assert kpack.pack_reversed(v, w) == rev, (coeffs, b, w)
        assert kpack.pack_negated(v, w) == neg, (coeffs, b, w)
        assert kpack.pack_negated_reversed(v, w) == nrev, (coeffs, b, w)
        n += 1
    assert n >= 200


def test_pack_kats(kpack):
    # pkg/tests/test_pack.py:26-59
    from paper_0712_4046_b200.kstypes import CoeffVec
    assert kpack.pack(CoeffVec((1, 2, 3), 8), 8) == 197121
    assert kpack.pack_reversed(CoeffVec((1, 2, 3), 8), 8) == 66051
    assert kpack.pack_negated(CoeffVec((3, 2, 1), 4), 4) == 227
    assert kpack.pack_negated_reversed(CoeffVec((3, 2, 1), 4), 4) == 737


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_pack_batched_vs_oracle(kpack, kind):
    from paper_0712_4046_b200.words import ints_to_words, words_to_ints
    rng = random.Random(40 + kind)
    fn = {0: O.pack, 1: O.pack_negated, 2: O.pack_reversed, 3: O.pack_negated_reversed}[kind]
    for L, b, w in [(1, 7, 4), (2, 64, 32), (255, 64, 34), (256, 64, 136), (1024, 32, 19), (333, 100, 51),
                    (4096, 128, 67)]:
        vecs = [[rng.randrange(1 << b) for _ in range(L)] for _ in range(9)]
        vecs[0] = [(1 << b) - 1] * L
        words = (b + 31) // 32
        arr = np.stack([ints_to_words(v, words) for v in vecs])
        out, meta = kpack.pack_batch(kind, arr, w, b)
        for i, v in enumerate(vecs):
            want = fn(v, w, b)
            mag = words_to_ints(out[i][None, :])[0]
            assert (-mag if meta[i, 0] else mag) == want, (L, b, w, i)
            assert meta[i, 1] == abs(want).bit_length()


def test_pack_errors(kpack):
    from paper_0712_4046_b200.kstypes import CoeffVec
    with pytest.raises(ValueError):
        kpack.pack(CoeffVec((1, 2), 9), 4)  # 2w < b (pack.py:55-59)
    bad = np.array([[[1 << 10], [3]]], dtype=np.uint32)
    with pytest.raises(ValueError):
        kpack.pack_batch(0, bad, 10, 10)  # coefficient >= 2^b, latched on the device
