"""The drop-in's domain equals the reference's: any coefficient bound
(pack.py:36-46, ksint.py:82-98).  Widths past the fast finish / register
reconstruction budgets (b >~ 490 bits) run through kmx_wide.cu; results are
bit-exact against the oracle (Python ints) for every variant, through the
drop-in entry points and the batched device API, plus the standalone
reconstruction at wide digit widths."""
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


@pytest.mark.parametrize("b", [490, 500, 545, 1000, 4096])
def test_dropin_wide_coefficients(kmx, b):
    rng = random.Random(b)
    fns = (kmx.ks1_mul, kmx.ks2_mul, kmx.ks3_mul, kmx.ks4_mul)
    for lf, lg in [(1, 1), (2, 2), (5, 3), (17, 17), (64, 40)]:
        f = [rng.randrange(1 << b) for _ in range(lf)]
        g = [rng.randrange(1 << b) for _ in range(lg)]
        f[0] = (1 << b) - 1
        want = O.ks_mul(1, f, g, b, mode="native")
        for fn in fns:
            got = fn(kmx.CoeffVec(tuple(f), b), kmx.CoeffVec(tuple(g), b))
            assert list(got.coeffs) == want, (fn.__name__, b, lf, lg)
    assert kmx.derive_params(2, 2, 500).width_full == 1001


@pytest.mark.parametrize("b", [600, 2048])
def test_batched_wide(kmx, b):
    from paper_0712_4046_b200.words import ints_to_words, words_to_ints
    rng = random.Random(7 * b)
    B, n = 5, 33
    w = (b + 31) // 32
    fs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    fs[1] = [(1 << b) - 1] * n
    gs[1] = [(1 << b) - 1] * n
    fd = torch.from_numpy(np.stack([ints_to_words(f, w) for f in fs]).view(np.int32)).cuda()
    gd = torch.from_numpy(np.stack([ints_to_words(g, w) for g in gs]).view(np.int32)).cuda()
    want = [O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in range(B)]
    for v in (1, 2, 3, 4):
        kb = kmx.KsBatch(v, B, n, n, b)
        h = kb(fd, gd)
        kb.status()
        a = h.cpu().numpy().view(np.uint32)
        assert [words_to_ints(a[p]) for p in range(B)] == want, v


@pytest.mark.parametrize("width", [545, 600, 2000])
def test_reconstruct_wide(kmx, width):
    rng = random.Random(width)
    for count in (1, 2, 9):
        top = (1 << width) * ((1 << width) - 1)
        vals = [rng.randrange(top) for _ in range(count)]
        vals[0] = top - 1
        fv = sum(h << (i * width) for i, h in enumerate(vals))
        rv = sum(h << ((count - 1 - i) * width) for i, h in enumerate(vals))
        m = (1 << width) - 1
        fwd = [(fv >> (i * width)) & m for i in range(count + 1)]
        rev = [(rv >> (i * width)) & m for i in range(count + 1)][::-1]
        got, fc, rc = kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(fwd), tuple(rev), width), with_carries=True)
        want, wfc, wrc = O.reconstruct(fwd, rev, width)
        assert list(got.coeffs) == want == vals
        assert fc == wfc and rc == wrc
    # inconsistent streams raise, as the reference does (ksint.py:157-177)
    bad = list(fwd)
    bad[-1] ^= 1
    with pytest.raises(kmx.ReconstructionError):
        kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(bad), tuple(rev), width))


@pytest.mark.parametrize("cbits", [31, 40, 100])
def test_bivariate_wide_coefficients(kmx, cbits):
    # bks_* over Z takes any integers (bipoly.py:53-56): 40-bit and wider
    # signed grids run through kmx_bks_wide_mul, bit-exact vs the schoolbook
    rng = random.Random(cbits)
    Z = kmx.ring_z()
    fns = (kmx.bks_standard, kmx.bks_reciprocal, kmx.bks_negated, kmx.bks_four)
    for lx, ly in [(1, 1), (2, 3), (5, 4), (9, 9)]:
        lim = 1 << cbits
        f = [[rng.randrange(-lim + 1, lim) for _ in range(ly)] for _ in range(lx)]
        g = [[rng.randrange(-lim + 1, lim) for _ in range(ly)] for _ in range(lx)]
        f[0][0] = lim - 1
        g[-1][-1] = -(lim - 1)
        want = O.schoolbook_bivar(f, g)
        F, Gp = kmx.BiPoly(tuple(map(tuple, f))), kmx.BiPoly(tuple(map(tuple, g)))
        for fn in fns:
            assert [list(r) for r in fn(F, Gp, Z).coeffs] == want, (fn.__name__, cbits, lx, ly)


def test_bivariate_int64_overflow_routes_wide(kmx):
    # 30-bit coefficients on a 64x64 grid overflow int64 accumulation: the
    # narrow kernel refuses (KMX_EINVAL) and the drop-in takes the wide path
    rng = random.Random(3)
    lx = ly = 24
    f = [[rng.randrange(-(1 << 29), 1 << 29) for _ in range(ly)] for _ in range(lx)]
    g = [[rng.randrange(-(1 << 29), 1 << 29) for _ in range(ly)] for _ in range(lx)]
    want = O.schoolbook_bivar(f, g)
    got = kmx.bks_four(kmx.BiPoly(tuple(map(tuple, f))), kmx.BiPoly(tuple(map(tuple, g))), kmx.ring_z())
    assert [list(r) for r in got.coeffs] == want
