"""GPU parity of the (Z/nZ)[x] front end (kmx_mod_mul: the KS path + K9
modular reduction) against fixtures generated from the reference's
kronmul.modpoly.mod_mul and against the oracle.  Bit-exact."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ks_oracle as O  # noqa: E402
from tests import golden_io as G  # noqa: E402

pytestmark = pytest.mark.gpu

CASES, TABLE = G.mod_golden()


@pytest.fixture(scope="module")
def mp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_0712_4046_b200 import modpoly
    return modpoly


def test_dropin_mod_golden(mp):
    for tag, f, g, n, h, counts in CASES:
        F, Gp = mp.ModPoly(tuple(f), n), mp.ModPoly(tuple(g), n)
        for v in (mp.Variant.KS1, mp.Variant.KS2, mp.Variant.KS3, mp.Variant.KS4, mp.Variant.AUTO):
            got = mp.mod_mul(F, Gp, v)
            assert list(got.coeffs) == h, (tag, v)
            assert got.modulus == n


def test_dropin_mod_stats(mp):
    # pkg/tests/test_modpoly.py:89-106: classical-mode limb products
    from paper_0712_4046_b200 import MulConfig, MulStats
    for tag, f, g, n, h, counts in CASES:
        if not counts:
            continue
        F, Gp = mp.ModPoly(tuple(f), n), mp.ModPoly(tuple(g), n)
        for i, v in enumerate((mp.Variant.KS1, mp.Variant.KS2, mp.Variant.KS3, mp.Variant.KS4)):
            s = MulStats()
            mp.mod_mul(F, Gp, v, stats=s, config=MulConfig(classical_only=True))
            assert s.limb_products == counts[f"ks{i + 1}"], (tag, v)


def test_mod_errors(mp):
    # pkg/tests/test_modpoly.py:39-44
    with pytest.raises(ValueError):
        mp.mod_mul(mp.ModPoly((1,), 5), mp.ModPoly((1,), 7))
    assert mp.mod_mul(mp.ModPoly((1,), 2), mp.ModPoly((1,), 2)).coeffs == (1,)
    # device-side range check (ModPoly invariant, modpoly.py:57-58) on the batched path
    f = torch.tensor([[1, 2, 7]], dtype=torch.int64, device="cuda")
    g = torch.tensor([[3, 4, 5]], dtype=torch.int64, device="cuda")
    op = mp.ModMulBatch(4, 1, 3, 3, 7, device="cuda")
    op(f, g)
    with pytest.raises(ValueError):
        op.status()
    with pytest.raises(ValueError):
        mp.mod_mul_host(1, np.array([[9]], dtype=np.uint64), np.array([[1]], dtype=np.uint64), 5)


@pytest.mark.parametrize("n", [13, 1009, (1 << 48) - 59, (1 << 64) - 59, 1 << 63, 2])
def test_mod_batch_against_oracle(mp, n):
    rng = random.Random(n % 1000003)
    B, lf, lg = 24, 300, 211
    fi = [[rng.randrange(n) for _ in range(lf)] for _ in range(B)]
    gi = [[rng.randrange(n) for _ in range(lg)] for _ in range(B)]
    fd = torch.from_numpy(np.array(fi, dtype=np.uint64).view(np.int64)).cuda()
    gd = torch.from_numpy(np.array(gi, dtype=np.uint64).view(np.int64)).cuda()
    outs = []
    for v in (1, 2, 3, 4):
        op = mp.ModMulBatch(v, B, lf, lg, n, device="cuda")
        h = op(fd, gd)
        op.status()
        outs.append(h.cpu().numpy().view(np.uint64))
    for v in range(1, 4):
        assert np.array_equal(outs[0], outs[v]), v
    for p in (0, B // 2, B - 1):
        want = O.mod_mul(1, fi[p], gi[p], n, mode="native")
        assert [int(x) for x in outs[3][p]] == want, p


def test_mod_host_batch_paper_sizes(mp):
    # the paper's section-4 experiment: 4-bit and 48-bit moduli
    rng = np.random.default_rng(4)
    for n, L in ((13, 2048), ((1 << 48) - 59, 1024)):
        f = rng.integers(0, n, size=(16, L), dtype=np.uint64)
        g = rng.integers(0, n, size=(16, L), dtype=np.uint64)
        want = None
        for v in (1, 2, 3, 4):
            h = mp.mod_mul_host(v, f, g, n)
            if want is None:
                want = [O.mod_mul(1, [int(x) for x in f[p]], [int(x) for x in g[p]], n, mode="native")
                        for p in (0, 15)]
            assert [int(x) for x in h[0]] == want[0] and [int(x) for x in h[15]] == want[1], (n, v)
