"""The reference's acceptance legs (pkg/tests/test_acceptance.py) on the GPU
path, through the batched C ABI.

  * exhaustive lengths 1..3 with coefficients < 8 (266,304 pairs, :43-55),
    grouped by (len_f, len_g) into one batched call per shape and variant;
  * 10^4 randomized cases, b <= 64, lengths log-uniform up to 64/256/512,
    mostly unequal (:57-76; the same generator, seed 101);
  * 10^4 reconstruction round trips, widths 2..128 (:154-173);
  * the bivariate equivalence over Z and Z/7 (:79-117; 1000 cases).
Every product is compared with an exact schoolbook (numpy or Python ints).
"""
import itertools
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


def log_uniform(rng, hi):
    return max(1, int(hi ** rng.random()))


def test_exhaustive_small_lengths(kmx):
    # the reference's leg pairs vectors of equal length (266,304 pairs); the
    # unequal-length combinations are checked too (74,752 more)
    checked = equal = 0
    for lf, lg in itertools.product((1, 2, 3), repeat=2):
        F = np.array(list(itertools.product(range(8), repeat=lf)), dtype=np.int64)
        G = np.array(list(itertools.product(range(8), repeat=lg)), dtype=np.int64)
        # every (f, g) combination: batch = 8^lf * 8^lg pairs
        fb = np.repeat(F, len(G), axis=0)
        gb = np.tile(G, (len(F), 1))
        want = np.zeros((len(fb), lf + lg - 1), dtype=np.int64)
        for i in range(lf):
            for j in range(lg):
                want[:, i + j] += fb[:, i] * gb[:, j]
        fw = np.ascontiguousarray(fb.astype(np.uint32)[:, :, None])
        gw = np.ascontiguousarray(gb.astype(np.uint32)[:, :, None])
        for v in (1, 2, 3, 4):
            h = kmx.ks_mul_host(v, fw, gw, 3)
            assert h.shape[2] == 1
            assert np.array_equal(h[:, :, 0].astype(np.int64), want), (lf, lg, v)
        checked += len(fb)
        equal += len(fb) if lf == lg else 0
    assert equal == 266304 and checked == 341056


def test_randomized_10k(kmx):
    rng = random.Random(101)
    unequal = 0
    for i in range(10_000):
        bound = rng.randrange(1, 65)
        hi = (64, 256, 512)[i % 3]
        lf, lg = log_uniform(rng, hi), log_uniform(rng, hi)
        unequal += lf != lg
        f = [rng.randrange(1 << bound) for _ in range(lf)]
        g = [rng.randrange(1 << bound) for _ in range(lg)]
        w = (bound + 31) // 32
        from paper_0712_4046_b200.words import ints_to_words, words_to_ints
        fw, gw = ints_to_words(f, w)[None], ints_to_words(g, w)[None]
        want = O.ks_mul(1, f, g, bound, mode="native")
        for v in (1, 2, 3, 4):
            h = kmx.ks_mul_host(v, fw, gw, bound, tune=False)
            assert words_to_ints(h[0]) == want, (i, v, bound, lf, lg)
    assert unequal > 1000


def test_reconstruction_round_trip_10k(kmx):
    rng = random.Random(303)
    for case in range(10_000):
        width = rng.randrange(2, 129)
        count = log_uniform(rng, 128)
        top = (1 << width) * ((1 << width) - 1)
        values = [rng.randrange(top) for _ in range(count)]
        fv = sum(h << (i * width) for i, h in enumerate(values))
        rv = sum(h << ((count - 1 - i) * width) for i, h in enumerate(values))
        mask = (1 << width) - 1
        fwd = tuple((fv >> (i * width)) & mask for i in range(count + 1))
        rev = tuple((rv >> ((count - i) * width)) & mask for i in range(count + 1))
        got, fc, rc = kmx.reconstruct_overlapped(kmx.OverlapDigits(fwd, rev, width), with_carries=True)
        assert list(got.coeffs) == values, (width, count, case)
        assert set(fc) <= {0, 1} and set(rc) <= {0, 1}


def test_bivariate_equivalence_1000(kmx):
    rings = [("Z", kmx.ring_z(), lambda r: r.randrange(-99, 100), None),
             ("Z/7", kmx.ring_zmod(7), lambda r: r.randrange(7), 7)]
    funcs = (kmx.bks_standard, kmx.bks_reciprocal, kmx.bks_negated, kmx.bks_four)
    rng = random.Random(202)
    cases = 0
    for _ in range(500):
        for name, ring, draw, n in rings:
            lx, ly = rng.randrange(1, 9), rng.randrange(1, 9)
            f = [[draw(rng) for _ in range(ly)] for _ in range(lx)]
            g = [[draw(rng) for _ in range(ly)] for _ in range(lx)]
            want = O.schoolbook_bivar(f, g)
            if n:
                want = [[c % n for c in row] for row in want]
            F, Gp = kmx.BiPoly(tuple(map(tuple, f))), kmx.BiPoly(tuple(map(tuple, g)))
            for fn in funcs:
                assert [list(r) for r in fn(F, Gp, ring).coeffs] == want, (name, fn.__name__, f, g)
            cases += 1
    assert cases >= 1000
    p = kmx.BiPoly(((1, 2), (3, 4)))
    for k in (1, 3, 10):
        for fn in (kmx.bks_negated, kmx.bks_four):
            with pytest.raises(kmx.MissingHalveError):
                fn(p, p, kmx.ring_zmod(2 ** k))


def test_random_medium_lengths(kmx):
    # beyond the reference's leg (lengths <= 512): lengths 300..3000, mostly unequal, widths
    # on both sides of the one- and two-word digit boundaries, signed and unsigned, small
    # batches -- the shapes on which the kernel selection changes (pair / cluster / per-stream
    # reconstruction, one- and two-window tensor-core tiles, warp / block / streaming packs);
    # the first and the last pair of every batch against an exact product, all variants equal
    from paper_0712_4046_b200.words import ints_to_words, words_to_ints
    rng = random.Random(20260)
    for case in range(48):
        signed = case % 4 == 0
        b = 32 if signed else rng.choice((5, 16, 27, 32, 33, 47, 64, 65, 96, 130))
        lf = rng.randrange(300, 3000)
        lg = lf if case % 5 == 0 else rng.randrange(300, 3000)
        B = rng.choice((1, 2, 3, 5))
        lo, hi = (-(1 << 31), 1 << 31) if signed else (0, 1 << b)
        fs = [[rng.randrange(lo, hi) for _ in range(lf)] for _ in range(B)]
        gs = [[rng.randrange(lo, hi) for _ in range(lg)] for _ in range(B)]
        if case % 7 == 0:  # extremes in one pair
            fs[-1] = [hi - 1] * lf
            gs[-1] = [lo if signed else hi - 1] * lg
        words = 1 if signed else (b + 31) // 32
        fd = torch.from_numpy(np.stack([ints_to_words(f, words, signed=signed) for f in fs]).view(np.int32)).cuda()
        gd = torch.from_numpy(np.stack([ints_to_words(g, words, signed=signed) for g in gs]).view(np.int32)).cuda()
        want = {}
        for p in {0, B - 1}:
            want[p] = (O.ks_mul_signed(1, fs[p], gs[p], b, mode="native") if signed
                       else O.ks_mul(1, fs[p], gs[p], b, mode="native"))
        first = None
        for v in (1, 2, 3, 4):
            kb = kmx.KsBatch(v, B, lf, lg, b, signed=signed)
            h = kb(fd, gd)
            kb.status()
            a = h.cpu().numpy().view(np.uint32)
            for p, w in want.items():
                assert words_to_ints(a[p], signed=signed) == w, (case, v, lf, lg, b, signed, p)
            if first is None:
                first = a
            else:
                assert np.array_equal(first, a), (case, v, lf, lg, b, signed)
