"""GPU parity of the bivariate reductions over Z/nZ (kmx_bks_mod_mul:
evaluation mod n, univariate products through the integer KS path, modular
half-sums and overlap recovery) against fixtures generated from the
reference's bks_* with ring_zmod(n), and against the oracle."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ks_oracle as O  # noqa: E402
from tests import golden_io as G  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kmx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_0712_4046_b200 as k
    return k


def test_dropin_bivar_mod_golden(kmx):
    fns = {1: kmx.bks_standard, 2: kmx.bks_reciprocal, 3: kmx.bks_negated, 4: kmx.bks_four}
    for n, f, g, h, missing in G.bivar_mod_cases():
        ring = kmx.ring_zmod(n)
        F = kmx.BiPoly(tuple(map(tuple, f)))
        Gp = kmx.BiPoly(tuple(map(tuple, g)))
        for v, fn in fns.items():
            if v in missing:
                with pytest.raises(kmx.MissingHalveError):
                    fn(F, Gp, ring)
                continue
            got = fn(F, Gp, ring)
            assert [list(r) for r in got.coeffs] == h, (n, v)


@pytest.mark.parametrize("n", [1009, (1 << 61) - 1, (1 << 64) - 59, 1 << 40])
def test_bivar_mod_batch_against_oracle(kmx, n):
    rng = random.Random(n % 99991)
    B, lx, ly = 6, 24, 17
    fs = [[[rng.randrange(n) for _ in range(ly)] for _ in range(lx)] for _ in range(B)]
    gs = [[[rng.randrange(n) for _ in range(ly)] for _ in range(lx)] for _ in range(B)]
    fd = torch.from_numpy(np.array(fs, dtype=np.uint64).view(np.int64)).cuda()
    gd = torch.from_numpy(np.array(gs, dtype=np.uint64).view(np.int64)).cuda()
    variants = (1, 2, 3, 4) if n % 2 else (1, 2)
    outs = []
    for v in variants:
        op = kmx.BksModBatch(v, B, lx, ly, n, device="cuda")
        h = op(fd, gd)
        op.status()
        outs.append(h.cpu().numpy().view(np.uint64))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    for p in (0, B - 1):
        want = O.bks_mod(1, fs[p], gs[p], n, umul=O.convolve_exact)
        assert [[int(x) for x in r] for r in outs[-1][p]] == want


def test_bivar_mod_errors(kmx):
    with pytest.raises(ValueError):
        kmx.BksModBatch(3, 1, 4, 4, 16, device="cuda")   # even n: no halving for the negated variant
    op = kmx.BksModBatch(1, 1, 2, 2, 7, device="cuda")
    f = torch.tensor([[[1, 2], [3, 9]]], dtype=torch.int64, device="cuda")   # 9 >= 7
    g = torch.tensor([[[1, 2], [3, 4]]], dtype=torch.int64, device="cuda")
    op(f, g)
    with pytest.raises(ValueError):
        op.status()
