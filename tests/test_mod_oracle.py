"""Pins the (Z/nZ)[x] oracle restatement (oracle/ks_oracle.py mod_mul,
schoolbook_mod, choose_variant) to fixtures generated from the reference's
kronmul.modpoly (tests/golden/make_golden_mod.py), and checks the host-side
mirror of the reference interface (paper_0712_4046_b200.modpoly: ModPoly
validation, choose_variant bands) without a GPU."""
import pytest

from oracle import ks_oracle as O
from tests import golden_io as G

CASES, TABLE = G.mod_golden()


def test_mod_oracle_against_reference_fixtures():
    for tag, f, g, n, h, counts in CASES:
        for v in (1, 2, 3, 4, 0):
            assert O.mod_mul(v, f, g, n, mode="native") == h, (tag, v)
        if len(f) * len(g) <= 40000:
            assert O.schoolbook_mod(f, g, n) == h, tag


def test_mod_oracle_classical_counts():
    # pkg/tests/test_modpoly.py:89-106 (classical-only limb products)
    for tag, f, g, n, h, counts in CASES:
        if not counts:
            continue
        for v in (1, 2, 3, 4):
            st = O.Counter()
            O.mod_mul(v, f, g, n, mode="karatsuba", stats=st, classical_only=True)
            assert st.limb_products == counts[f"ks{v}"], (tag, v)
        assert counts["ks1"] > 2 * counts["ks4"]


def test_worked_example_mod():
    # pkg/tests/test_modpoly.py:29-36
    f, g = [274, 610, 887, 621], [553, 298, 424, 790]
    want = [151522, 418982, 788467, 82836, 43043, 964034, 490590]
    for v in (0, 1, 2, 3, 4):
        assert O.mod_mul(v, f, g, 1000003) == want


def test_choose_variant_table_matches_reference():
    from paper_0712_4046_b200.modpoly import Variant, choose_variant
    for L, bits, want in TABLE:
        assert choose_variant(L, bits).value == want
        assert {1: "ks1", 3: "ks3", 4: "ks4"}[O.choose_variant(L, bits)] == want
    # pkg/tests/test_modpoly.py:80-87
    from paper_0712_4046_b200.modpoly import AutoThresholds
    custom = AutoThresholds(ks1_max_length=2, ks3_max_length=4)
    assert choose_variant(3, 10, custom) is Variant.KS3
    assert choose_variant(5, 10, custom) is Variant.KS4
    with pytest.raises(ValueError):
        choose_variant(0, 3)


def test_modpoly_validation():
    # pkg/tests/test_modpoly.py:18-26
    from paper_0712_4046_b200.modpoly import ModPoly
    with pytest.raises(ValueError):
        ModPoly((0,), 1)
    with pytest.raises(ValueError):
        ModPoly((), 5)
    with pytest.raises(ValueError):
        ModPoly((5,), 5)
    with pytest.raises(ValueError):
        ModPoly((0,), 1 << 65)
    assert ModPoly((1, 2), 3).coeffs == (1, 2)
