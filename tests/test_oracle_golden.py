"""Pins the CPU oracle (oracle/ks_oracle.py) to the reference: every golden
vector generated from the reference package (tests/golden/make_golden.py) and
the reference's own known-answer tests (pkg/tests/test_ksint.py,
test_pack.py, test_bipoly.py, test_base10_example.py) must reproduce."""
import random

import pytest

from oracle import ks_oracle as O
from tests import golden_io as G

KS_CASES = G.ks_cases()


def test_reference_worked_example():
    # pkg/tests/test_ksint.py:12-14, :59-61
    f, g = [274, 610, 887, 621], [553, 298, 424, 790]
    want = [151522, 418982, 788467, 1082839, 1043046, 964034, 490590]
    for v in (1, 2, 3, 4):
        assert O.ks_mul(v, f, g, 10) == want


def test_reference_param_kats():
    # pkg/tests/test_ksint.py:24-33
    p = O.derive_params(4, 4, 10)
    assert (p.e, p.n1, p.n2, p.n4) == (2, 22, 11, 6)
    assert O.derive_params(1, 1, 7).e == 0 and O.derive_params(1, 1, 7).n1 == 14
    assert O.derive_params(5, 3, 7).e == 2
    with pytest.raises(ValueError):
        O.derive_params(0, 1, 4)


def test_reference_pack_kats():
    # pkg/tests/test_pack.py:26-59
    assert O.pack([1, 2, 3], 8, 8) == 197121
    assert O.pack_reversed([1, 2, 3], 8, 8) == 66051
    assert O.pack_negated([3, 2, 1], 4, 4) == 227
    assert O.pack_negated_reversed([3, 2, 1], 4, 4) == 737
    assert O.pack_negated_reversed([11], 4, 4) == 11
    with pytest.raises(ValueError):
        O.pack([255], 3, 8)


def test_reference_reconstruction_kats():
    # pkg/tests/test_ksint.py:115-127
    assert O.reconstruct([5, 2], [2, 5], 3)[0] == [21]
    h, fc, rc = O.reconstruct([3, 3, 7, 0], [0, 4, 3, 6], 3)
    assert h == [3, 11, 6] and fc == [0, 0, 0, 0] and rc == [0, 0, 0]


def test_reference_base10_four_point_intermediates():
    # pkg/tests/test_base10_example.py:98-136, restated at binary width:
    # the half-sums are the two overlapped packings of the even/odd parts.
    f, g = [274, 610, 887, 621], [553, 298, 424, 790]
    h = O.schoolbook(f, g)
    n = 6
    pf = O.pack(f, n, 10) * O.pack(g, n, 10)
    pn = O.pack_negated(f, n, 10) * O.pack_negated(g, n, 10)
    w = 2 * n
    assert O.halve_exact(pf + pn) == sum(c << (w * i) for i, c in enumerate(h[0::2]))
    assert O.shr_exact(O.halve_exact(pf - pn), n) == sum(c << (w * i) for i, c in enumerate(h[1::2]))


@pytest.mark.parametrize("idx", range(0, len(KS_CASES)))
def test_oracle_matches_reference_golden(idx):
    tag, f, g, b, h = KS_CASES[idx]
    mode = "native" if len(f) > 1000 else "karatsuba"
    for v in (1, 2, 3, 4):
        assert O.ks_mul(v, f, g, b, mode=mode) == h, (tag, v)


def test_oracle_pack_golden():
    for c, b, w, pk, rv, ng, nr in G.pack_cases():
        assert O.pack(c, w, b) == pk
        assert O.pack_reversed(c, w, b) == rv
        assert O.pack_negated(c, w, b) == ng
        assert O.pack_negated_reversed(c, w, b) == nr


def test_oracle_reconstruction_golden():
    for fwd, rev, w, h in G.recon_cases():
        assert O.reconstruct(fwd, rev, w)[0] == h


def test_oracle_rejects_out_of_range_reconstruction():
    # pkg/tests/test_ksint.py:157-162
    w = 4
    top = (1 << w) * ((1 << w) - 1)
    vals = [top, 3]
    fv = sum(h << (i * w) for i, h in enumerate(vals))
    rv = sum(h << ((1 - i) * w) for i, h in enumerate(vals))
    m = (1 << w) - 1
    fwd = [(fv >> (i * w)) & m for i in range(3)]
    rev = [(rv >> (i * w)) & m for i in range(3)][::-1]
    with pytest.raises(O.OracleReconstructionError):
        O.reconstruct(fwd, rev, w)


def test_oracle_signed_golden():
    for f, g, h in G.signed_cases():
        for v in (1, 2, 3, 4):
            assert O.ks_mul_signed(v, f, g, 32) == h


def test_oracle_bivariate_golden():
    for tag, f, g, h in G.bivar_cases():
        for v in (1, 2, 3, 4):
            assert O.bks(v, f, g) == h, (tag, v)
        if len(f) <= 8:
            assert O.schoolbook_bivar(f, g) == h


def test_oracle_limb_stats_law():
    # bignat.py:327-330: classical counts limbs(x)*limbs(y); the acceptance
    # work ratio (pkg/tests/test_acceptance.py:176-192) must hold.
    top = (1 << 48) - 1
    f = g = [top] * 256
    counts = {}
    for v in (1, 2, 3, 4):
        c = O.Counter()
        O.ks_mul(v, f, g, 48, stats=c, classical_only=True)
        counts[v] = c.limb_products
    assert counts == {1: 173056, 2: 86528, 3: 86528, 4: 44100}


def test_words_roundtrip():
    rng = random.Random(3)
    vals = [[rng.randrange(1 << 100) for _ in range(5)] for _ in range(3)]
    assert O.words_to_ints(O.ints_to_words(vals, 4)) == vals
    sv = [-5, 7, -(1 << 70)]
    w = O.ints_to_words(sv, 3, signed=True)
    back = [v - (1 << 96) if v >> 95 else v for v in O.words_to_ints(w)]
    assert back == sv


def test_oracle_uni_schoolbook_matches_convolution():
    # the restated reference UniMul (oracle.py:58-69) used by the CPU baseline
    rng = random.Random(9)
    for _ in range(20):
        a = [rng.randrange(-99, 100) for _ in range(rng.randrange(1, 30))]
        b = [rng.randrange(-99, 100) for _ in range(rng.randrange(1, 30))]
        assert O.uni_schoolbook(a, b) == O.convolve_exact(a, b) == O.schoolbook(a, b)
    tag, f, g, h = G.bivar_cases()[3]
    assert O.bks(4, f, g, umul=O.uni_schoolbook) == h


def test_mul_count_follows_the_reference_recursion():
    """ksint._mul_count (host: operand lengths of the Karatsuba recursion,
    bignat.py:344-371) against the oracle's counted multiply on random and
    all-ones operands, default and small thresholds."""
    import random
    from paper_0712_4046_b200.ksint import _mul_count
    from paper_0712_4046_b200.kstypes import MulConfig
    rng = random.Random(5)
    for bits_x, bits_y in ((64, 64), (1024, 1024), (1100, 5000), (4096, 4000), (20000, 20000), (7, 30000)):
        for x, y in ((rng.getrandbits(bits_x) | 1 << (bits_x - 1), rng.getrandbits(bits_y) | 1 << (bits_y - 1)),
                     ((1 << bits_x) - 1, (1 << bits_y) - 1)):
            for thr in (16, 2):
                st = O.Counter()
                O.mul(x, y, "karatsuba", st, threshold=thr)
                assert _mul_count(x, y, MulConfig(karatsuba_threshold=thr)) == st.limb_products
            st = O.Counter()
            O.mul(x, y, "karatsuba", st, classical_only=True)
            assert _mul_count(x, y, MulConfig(classical_only=True)) == st.limb_products


def test_oracle_stats_golden():
    """The oracle's counted multiply against MulStats values the reference
    reported (default MulConfig and classical_only; tests/golden/make_golden_stats.py)."""
    for f, g, b, counts in G.stats_cases():
        for name, kw in (("default", {}), ("classical", {"classical_only": True})):
            row = []
            for v in (1, 2, 3, 4):
                c = O.Counter()
                O.ks_mul(v, f, g, b, stats=c, **kw)
                row.append(c.limb_products)
            assert row == counts[name], (len(f), len(g), b, name)
