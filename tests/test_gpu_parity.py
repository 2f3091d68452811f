"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Bit-exact for every case (integer path)."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ks_oracle as O  # noqa: E402
from tests import golden_io as G  # noqa: E402

pytestmark = pytest.mark.gpu

KS_CASES = G.ks_cases()


@pytest.fixture(scope="module")
def kmx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_0712_4046_b200 as k
    return k


def _dev_words(vals_2d, words, signed=False):
    from paper_0712_4046_b200.words import ints_to_words
    arr = np.stack([ints_to_words(v, words, signed=signed) for v in vals_2d])
    return torch.from_numpy(arr.view(np.int32)).cuda()


def _host_ints(t, signed=False):
    from paper_0712_4046_b200.words import words_to_ints
    a = t.cpu().numpy().view(np.uint32)
    return [words_to_ints(a[p], signed=signed) for p in range(a.shape[0])]


# ----------------------------------------------------------- golden (drop-in)
@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_dropin_golden(kmx, variant):
    fn = {1: kmx.ks1_mul, 2: kmx.ks2_mul, 3: kmx.ks3_mul, 4: kmx.ks4_mul}[variant]
    for tag, f, g, b, h in KS_CASES:
        got = fn(kmx.CoeffVec(tuple(f), b), kmx.CoeffVec(tuple(g), b))
        assert list(got.coeffs) == h, (tag, variant)
        assert got.width_bound_bits == 2 * b + (min(len(f), len(g)) - 1).bit_length()


def test_dropin_worked_example_and_kats(kmx):
    # pkg/tests/test_ksint.py:12-14, :64-69
    F = kmx.CoeffVec((274, 610, 887, 621), 10)
    Gv = kmx.CoeffVec((553, 298, 424, 790), 10)
    H = (151522, 418982, 788467, 1082839, 1043046, 964034, 490590)
    for fn in (kmx.ks1_mul, kmx.ks2_mul, kmx.ks3_mul, kmx.ks4_mul):
        assert fn(F, Gv).coeffs == H
        assert fn(kmx.CoeffVec((0, 0, 0), 5), kmx.CoeffVec((7, 21, 30), 5)).coeffs == (0,) * 5
        assert fn(kmx.CoeffVec((9,), 4), kmx.CoeffVec((13,), 4)).coeffs == (117,)


def test_dropin_stats_match_reference_counts(kmx):
    # pkg/tests/test_acceptance.py:176-192 (classical counts, L=256, b=48)
    top = (1 << 48) - 1
    f = kmx.CoeffVec((top,) * 256, 48)
    cfg = kmx.MulConfig(classical_only=True)
    counts = {}
    for v, fn in enumerate((kmx.ks1_mul, kmx.ks2_mul, kmx.ks3_mul, kmx.ks4_mul), 1):
        st = kmx.MulStats()
        fn(f, f, stats=st, config=cfg)
        counts[v] = st.limb_products
    assert counts == {1: 173056, 2: 86528, 3: 86528, 4: 44100}


def test_dropin_stats_follow_mulconfig(kmx):
    # MulStats.limb_products for the default MulConfig (Karatsuba above 16 limbs),
    # karatsuba_threshold=2 and classical_only, against counts the reference
    # reported (tests/golden/make_golden_stats.py; bignat.py:323-371)
    cfgs = {"default": None, "thr2": kmx.MulConfig(karatsuba_threshold=2),
            "classical": kmx.MulConfig(classical_only=True)}
    for f, g, b, counts in G.stats_cases():
        F, Gv = kmx.CoeffVec(tuple(f), b), kmx.CoeffVec(tuple(g), b)
        for name, cfg in cfgs.items():
            got = []
            for fn in (kmx.ks1_mul, kmx.ks2_mul, kmx.ks3_mul, kmx.ks4_mul):
                st = kmx.MulStats()
                fn(F, Gv, stats=st, config=cfg)
                got.append(st.limb_products)
            assert got == counts[name], (len(f), len(g), b, name)


def test_dropin_reconstruct_golden(kmx):
    for fwd, rev, w, h in G.recon_cases():
        got = kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(fwd), tuple(rev), w))
        assert list(got.coeffs) == h
    got, fc, rc = kmx.reconstruct_overlapped(kmx.OverlapDigits((3, 3, 7, 0), (0, 4, 3, 6), 3),
                                             with_carries=True)
    assert got.coeffs == (3, 11, 6) and fc == [0, 0, 0, 0] and rc == [0, 0, 0]


def test_dropin_reconstruct_rejects(kmx):
    # pkg/tests/test_ksint.py:157-162
    w = 4
    top = (1 << w) * ((1 << w) - 1)
    vals = [top, 3]
    fv = sum(h << (i * w) for i, h in enumerate(vals))
    rv = sum(h << ((1 - i) * w) for i, h in enumerate(vals))
    m = (1 << w) - 1
    fwd = [(fv >> (i * w)) & m for i in range(3)]
    rev = [(rv >> (i * w)) & m for i in range(3)][::-1]
    with pytest.raises(kmx.ReconstructionError):
        kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(fwd), tuple(rev), w))


def test_dropin_reconstruct_long_streams(kmx):
    # streams of >= 256 digits of at most 64 bits take the one-CTA-per-pair
    # kernel (kmx_recon2.cu): round trips at both digit word counts, with 16-byte
    # aligned and unaligned stream slots, full and ragged last segments, the
    # extreme values, and the rejection of an inconsistent stream (ksint.py:137-179)
    rng = random.Random(11)
    for w, count in ((7, 256), (32, 300), (33, 257), (38, 1024), (50, 1001), (64, 513), (64, 2049), (19, 4100)):
        top = (1 << w) * ((1 << w) - 1)
        for kind in ("random", "max", "zero"):
            if kind == "random":
                vals = [rng.randrange(top) for _ in range(count)]
            elif kind == "max":
                vals = [top - 1] * count
            else:
                vals = [0] * count
            fv = sum(h << (i * w) for i, h in enumerate(vals))
            rv = sum(h << ((count - 1 - i) * w) for i, h in enumerate(vals))
            m = (1 << w) - 1
            fwd = [(fv >> (i * w)) & m for i in range(count + 1)]
            rev = [(rv >> (i * w)) & m for i in range(count + 1)][::-1]
            got = kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(fwd), tuple(rev), w))
            assert list(got.coeffs) == vals, (w, count, kind)
            if kind == "random":
                bad = list(fwd)
                bad[count // 2] ^= 1
                with pytest.raises(kmx.ReconstructionError):
                    kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(bad), tuple(rev), w))
        # a coefficient equal to 2^w (2^w - 1) is out of range (ksint.py:157-158)
        vals = [rng.randrange(top) for _ in range(count)]
        vals[count - 3] = top
        fv = sum(h << (i * w) for i, h in enumerate(vals))
        rv = sum(h << ((count - 1 - i) * w) for i, h in enumerate(vals))
        fwd = [(fv >> (i * w)) & m for i in range(count + 1)]
        rev = [(rv >> (i * w)) & m for i in range(count + 1)][::-1]
        with pytest.raises(kmx.ReconstructionError):
            kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(fwd), tuple(rev), w))


def test_dropin_random_reconstruct_carries(kmx):
    rng = random.Random(5)
    for _ in range(200):
        w = rng.randrange(2, 140)
        count = rng.randrange(1, 40)
        top = (1 << w) * ((1 << w) - 1)
        vals = [rng.randrange(top) for _ in range(count)]
        fv = sum(h << (i * w) for i, h in enumerate(vals))
        rv = sum(h << ((count - 1 - i) * w) for i, h in enumerate(vals))
        m = (1 << w) - 1
        fwd = [(fv >> (i * w)) & m for i in range(count + 1)]
        rev = [(rv >> (i * w)) & m for i in range(count + 1)][::-1]
        got, fc, rc = kmx.reconstruct_overlapped(kmx.OverlapDigits(tuple(fwd), tuple(rev), w),
                                                 with_carries=True)
        want, wfc, wrc = O.reconstruct(fwd, rev, w)
        assert list(got.coeffs) == want == vals
        assert fc == wfc and rc == wrc


def test_invalid_coefficient_raises(kmx):
    # batched path validates 0 <= c < 2^b on the device (pack.py:36-46)
    f = np.zeros((1, 4, 1), dtype=np.uint32)
    f[0, 2, 0] = 1 << 10
    with pytest.raises(ValueError):
        kmx.ks_mul_host(1, f, f.copy(), 10)


# --------------------------------------------------------- batched configs
def _check_batch(kmx, variant, fs, gs, b, want, signed=False):
    words = 1 if signed else (b + 31) // 32
    kb = kmx.KsBatch(variant, len(fs), len(fs[0]), len(gs[0]), b, signed=signed)
    h = kb(_dev_words(fs, words, signed), _dev_words(gs, words, signed))
    kb.status()
    got = _host_ints(h, signed=signed)
    for p, w in want.items():
        assert got[p] == w, (variant, p)
    return got


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_config1_batch64(kmx, variant):
    rng = random.Random(101)
    fs = [[rng.randrange(1 << 64) for _ in range(256)] for _ in range(64)]
    gs = [[rng.randrange(1 << 64) for _ in range(256)] for _ in range(64)]
    want = {p: O.ks_mul(1, fs[p], gs[p], 64, mode="native") for p in range(64)}
    _check_batch(kmx, variant, fs, gs, 64, want)


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_config2_signed(kmx, variant):
    rng = random.Random(202)
    B, n = 64, 1024
    fs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    fs[0] = [-2**31] * n
    gs[0] = [-2**31] * n
    want = {p: O.ks_mul_signed(1, fs[p], gs[p], 32, mode="native") for p in (0, 1, 17, 63)}
    _check_batch(kmx, variant, fs, gs, 32, want, signed=True)


@pytest.mark.parametrize("signed", [False, True])
def test_wider_output_records(kmx, signed):
    # a caller may ask for more words per coefficient than the minimum: the upper words are the
    # zero / sign extension (the coefficient writers of every finish / reconstruction kernel)
    rng = random.Random(303)
    B, lf, lg, b = 3, 700, 640, 32 if signed else 27
    if signed:
        fs = [[rng.randrange(-2**31, 2**31) for _ in range(lf)] for _ in range(B)]
        gs = [[rng.randrange(-2**31, 2**31) for _ in range(lg)] for _ in range(B)]
    else:
        fs = [[rng.randrange(1 << b) for _ in range(lf)] for _ in range(B)]
        gs = [[rng.randrange(1 << b) for _ in range(lg)] for _ in range(B)]
    words = 1
    fd, gd = _dev_words(fs, words, signed), _dev_words(gs, words, signed)
    for v in (1, 2, 3, 4):
        kb = kmx.KsBatch(v, B, lf, lg, b, signed=signed)
        base = _host_ints(kb(fd, gd), signed=signed)
        kb.status()
        kw = kmx.KsBatch(v, B, lf, lg, b, signed=signed)
        kw.out_words += 3
        wide = _host_ints(kw(fd, gd), signed=signed)
        kw.status()
        assert wide == base, (v, signed)


def test_signed_golden(kmx):
    for f, g, h in G.signed_cases():
        for v in (1, 2, 3, 4):
            kb = kmx.KsBatch(v, 1, len(f), len(g), 32, signed=True)
            out = kb(_dev_words([f], 1, True), _dev_words([g], 1, True))
            kb.status()
            assert _host_ints(out, signed=True)[0] == h


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_config4_pairs(kmx, variant):
    rng = random.Random(404)
    B, n, b = 4, 4096, 128
    fs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    want = {p: O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in (0, 3)}
    _check_batch(kmx, variant, fs, gs, b, want)


@pytest.mark.parametrize("n", [16, 64, 256, 1024])
@pytest.mark.parametrize("b", [8, 32, 64, 128, 256])
def test_config5_grid(kmx, n, b):
    rng = random.Random(n * 1000 + b)
    B = 3
    fs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    want = {p: O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in range(B)}
    for v in (1, 2, 3, 4):
        _check_batch(kmx, v, fs, gs, b, want)


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_unequal_and_edge_lengths(kmx, variant):
    rng = random.Random(variant)
    for lf, lg, b in [(1, 1, 1), (1, 7, 5), (7, 1, 64), (2, 300, 33), (513, 40, 17), (100, 101, 256),
                      (3, 2, 1), (1000, 3, 96)]:
        fs = [[rng.randrange(1 << b) for _ in range(lf)] for _ in range(2)]
        gs = [[rng.randrange(1 << b) for _ in range(lg)] for _ in range(2)]
        fs[1] = [(1 << b) - 1] * lf
        gs[1] = [(1 << b) - 1] * lg
        want = {p: O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in range(2)}
        _check_batch(kmx, variant, fs, gs, b, want)


def test_batch_zero_is_noop(kmx):
    kb = kmx.KsBatch(4, 0, 8, 8, 16)
    e = torch.empty((0, 8, 1), dtype=torch.int32, device="cuda")
    kb(e, e)


# ------------------------------------------------------------- bivariate
@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_bivariate_golden(kmx, variant):
    fn = {1: kmx.bks_standard, 2: kmx.bks_reciprocal, 3: kmx.bks_negated, 4: kmx.bks_four}[variant]
    Z = kmx.ring_z()
    for tag, f, g, h in G.bivar_cases():
        got = fn(kmx.BiPoly(tuple(map(tuple, f))), kmx.BiPoly(tuple(map(tuple, g))), Z)
        assert [list(r) for r in got.coeffs] == h, (tag, variant)


def test_bivariate_missing_halve(kmx):
    p = kmx.BiPoly(((1, 2), (3, 4)))
    for k in (1, 3, 10):
        for fn in (kmx.bks_negated, kmx.bks_four):
            with pytest.raises(kmx.MissingHalveError):
                fn(p, p, kmx.ring_zmod(2 ** k))


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_config3_batch(kmx, variant):
    rng = np.random.default_rng(303)
    B = 256
    f = rng.integers(0, 1 << 16, size=(B, 64, 64), dtype=np.int64).astype(np.int32)
    g = rng.integers(0, 1 << 16, size=(B, 64, 64), dtype=np.int64).astype(np.int32)
    bb = kmx.BksBatch(variant, B, 64, 64, 16)
    h = bb(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda())
    bb.status()
    hc = h.cpu().numpy()
    for p in (0, 255):
        want = O.bks(4, f[p].tolist(), g[p].tolist())
        assert hc[p].tolist() == want


# ------------------------------------------- size-independent checksums
def _eval_mod(coeffs_2d, x, p):
    # Horner evaluation of each row at x mod p (numpy object -> ints)
    out = []
    for row in coeffs_2d:
        acc = 0
        for c in reversed(row):
            acc = (acc * x + c) % p
        out.append(acc)
    return out


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_full_config2_checksum(kmx, variant):
    # every pair of the full BASELINE config-2 batch: h(x0) == f(x0) g(x0) mod p
    rng = np.random.default_rng(22)
    B, n = 1024, 1024
    f = rng.integers(-2**31, 2**31, size=(B, n, 1), dtype=np.int64).astype(np.int32)
    g = rng.integers(-2**31, 2**31, size=(B, n, 1), dtype=np.int64).astype(np.int32)
    kb = kmx.KsBatch(variant, B, n, n, 32, signed=True)
    h = kb(torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda())
    kb.status()
    hv = _host_ints(h, signed=True)
    p, x = (1 << 61) - 1, 1234567891011
    fe = _eval_mod(f[:, :, 0].tolist(), x, p)
    ge = _eval_mod(g[:, :, 0].tolist(), x, p)
    he = _eval_mod(hv, x, p)
    assert all((a * c - d) % p == 0 for a, c, d in zip(fe, ge, he))


@pytest.mark.parametrize("variant", [1, 4])
def test_host_pipelined_path(kmx, variant):
    # the host API splits large batches into chunks over several streams;
    # an uneven batch exercises the tail chunk
    rng = np.random.default_rng(77)
    B, n = 777, 1024
    f = rng.integers(-2**31, 2**31, size=(B, n, 1), dtype=np.int64).astype(np.int32).view(np.uint32)
    g = rng.integers(-2**31, 2**31, size=(B, n, 1), dtype=np.int64).astype(np.int32).view(np.uint32)
    fp = torch.from_numpy(f.view(np.int32)).pin_memory().numpy().view(np.uint32)
    gp = torch.from_numpy(g.view(np.int32)).pin_memory().numpy().view(np.uint32)
    h = kmx.ks_mul_host(variant, fp, gp, 32, signed=True)
    from paper_0712_4046_b200.words import words_to_ints
    for p in (0, 388, 776):
        want = O.ks_mul_signed(1, [int(x) for x in f[p, :, 0].view(np.int32)],
                               [int(x) for x in g[p, :, 0].view(np.int32)], 32, mode="native")
        assert words_to_ints(h[p], signed=True) == want


@pytest.mark.parametrize("n,b", [(8192, 8), (4096, 256), (8192, 64)])
def test_config5_large_points(kmx, n, b):
    # long digit streams (CTA reconstruction, thousands of steps) and large products
    rng = random.Random(n + b)
    fs = [[rng.randrange(1 << b) for _ in range(n)]]
    gs = [[rng.randrange(1 << b) for _ in range(n)]]
    want = {0: O.ks_mul(1, fs[0], gs[0], b, mode="native")}
    for v in (1, 2, 3, 4):
        _check_batch(kmx, v, fs, gs, b, want)


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_cuda_graph_replay(kmx, variant):
    # the bench replays a captured CUDA graph of the whole step; results must
    # match the oracle on every replay, including after new inputs are copied in
    rng = random.Random(55 + variant)
    B, n, b = 8, 256, 64
    fs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
    kb = kmx.KsBatch(variant, B, n, n, b)
    fd, gd = _dev_words(fs, 2), _dev_words(gs, 2)
    graph, out = kb.capture(fd, gd)
    for rep in range(2):
        graph.replay()
        kb.status()
        got = _host_ints(out)
        assert got[rep] == O.ks_mul(1, fs[rep], gs[rep], b, mode="native")
        fs2 = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
        fd.copy_(_dev_words(fs2, 2))
        fs = fs2
