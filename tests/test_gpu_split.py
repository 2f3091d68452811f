"""The split batch path (kmx_ks_mul over two streams, fork/join events) at
batches >= 256: bit-exact against the oracle on odd batch sizes, signed and
unsigned, eager and CUDA-graph-captured, with the device error flag and the
MulStats count aggregated over the parts."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ks_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kmx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_0712_4046_b200 as k
    return k


def _dev(vals, words, signed=False):
    from paper_0712_4046_b200.words import ints_to_words
    return torch.from_numpy(np.stack([ints_to_words(v, words, signed=signed) for v in vals]).view(np.int32)).cuda()


def _ints(t, signed=False):
    from paper_0712_4046_b200.words import words_to_ints
    a = t.cpu().numpy().view(np.uint32)
    return [words_to_ints(a[p], signed=signed) for p in range(a.shape[0])]


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_split_signed_odd_batch(kmx, variant):
    rng = random.Random(300 + variant)
    B, n = 301, 64
    fs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    fs[150] = [-2**31] * n
    gs[150] = [-2**31] * n
    kb = kmx.KsBatch(variant, B, n, n, 32, signed=True)
    h = kb(_dev(fs, 1, True), _dev(gs, 1, True))
    kb.status()
    got = _ints(h, signed=True)
    for p in (0, 149, 150, 151, 300):
        assert got[p] == O.ks_mul_signed(1, fs[p], gs[p], 32, mode="native"), p


@pytest.mark.parametrize("variant", [1, 4])
def test_split_graph_and_stats(kmx, variant):
    rng = random.Random(400 + variant)
    B, lf, lg, b = 257, 40, 23, 64
    fs = [[rng.randrange(1 << b) for _ in range(lf)] for _ in range(B)]
    gs = [[rng.randrange(1 << b) for _ in range(lg)] for _ in range(B)]
    kb = kmx.KsBatch(variant, B, lf, lg, b)
    fd, gd = _dev(fs, 2), _dev(gs, 2)
    graph, out = kb.capture(fd, gd)
    graph.replay()
    kb.status()
    got = _ints(out)
    for p in (0, 128, 129, 256):
        assert got[p] == O.ks_mul(1, fs[p], gs[p], b, mode="native"), p
    # MulStats classical count summed over the split parts (bignat.py:327-330)
    want = 0
    for p in range(B):
        st = O.Counter()
        O.ks_mul(variant, fs[p], gs[p], b, mode="karatsuba", stats=st, classical_only=True)
        want += st.limb_products
    assert kb.limb_products() == want


def test_split_error_flag(kmx):
    # an out-of-range coefficient in the second part must surface through the shared flag
    B, n, b = 300, 16, 20
    rng = random.Random(9)
    fs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    fs[299][3] = 1 << b
    kb = kmx.KsBatch(4, B, n, n, b)
    kb(_dev(fs, 1), _dev(gs, 1))
    with pytest.raises(ValueError):
        kb.status()
