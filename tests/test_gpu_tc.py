"""GPU parity of the tcgen05 multiply engine (kmx_tc.cu) against the CPU oracle
and against the integer-pipe engine (kmx_mul.cu), bit-exact.

The engine is chosen per call from the environment (KMX_TC=0 forces the
integer pipe; KMX_TC_H / KMX_TC_TPC / KMX_TC_KC force the tile width, the
tiles per CTA and the K-steps per B chunk), so one process covers every
tiling: single and split tile ranges (band spills at range boundaries),
double-buffered B chunks, and accumulators past 2^31 (all-ones operands)."""
import os
import random

import pytest

torch = pytest.importorskip("torch")

from oracle import ks_oracle as O  # noqa: E402
from tests.test_gpu_parity import _check_batch, _dev_words, _host_ints  # noqa: E402

pytestmark = pytest.mark.gpu

_KEYS = ("KMX_TC", "KMX_TC_H", "KMX_TC_TPC", "KMX_TC_KC", "KMX_FUSE")


@pytest.fixture(scope="module")
def kmx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_0712_4046_b200 as k
    return k


@pytest.fixture
def env():
    saved = {k: os.environ.get(k) for k in _KEYS}
    yield os.environ
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _cases(rng, shapes, pairs=2):
    for lf, lg, b in shapes:
        fs = [[rng.randrange(1 << b) for _ in range(lf)] for _ in range(pairs)]
        gs = [[rng.randrange(1 << b) for _ in range(lg)] for _ in range(pairs)]
        fs[-1] = [(1 << b) - 1] * lf
        gs[-1] = [(1 << b) - 1] * lg
        yield lf, lg, b, fs, gs


def test_engine_is_tensor_for_the_bench_shapes(kmx, env):
    env.pop("KMX_TC", None)
    # c2 (signed int32, n=1024) and c1 (u64, n=256) products run on tcgen05
    for v in (1, 2, 3, 4):
        assert kmx.mul_engine(v, 1024, 1024, 32, signed=True) == "tensor"
        assert kmx.mul_engine(v, 256, 256, 64) == "tensor"
    env["KMX_TC"] = "0"
    assert kmx.mul_engine(4, 1024, 1024, 32, signed=True) == "imad"


@pytest.mark.parametrize("H", [1, 2, 3, 4, 6, 8])
def test_forced_tile_widths(kmx, env, H):
    env["KMX_TC"] = "1"
    env["KMX_TC_H"] = str(H)
    rng = random.Random(900 + H)
    for lf, lg, b, fs, gs in _cases(rng, [(64, 64, 64), (1024, 1024, 32), (300, 17, 200), (5, 700, 96),
                                          (1500, 1500, 64)]):
        assert kmx.mul_engine(4, lf, lg, b) == "tensor"
        want = {p: O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in range(2)}
        for v in (1, 2, 3, 4):
            _check_batch(kmx, v, fs, gs, b, want)


@pytest.mark.parametrize("tpc,kc", [(1, 8), (2, 8), (1, 32), (3, 16)])
def test_split_tile_ranges_and_chunks(kmx, env, tpc, kc):
    # several CTAs per product: each range normalises its tiles and hands its
    # top carry to K3 as a band spill; small K-chunks cycle the B buffers
    env.update(KMX_TC="1", KMX_TC_TPC=str(tpc), KMX_TC_KC=str(kc), KMX_TC_H="1")
    rng = random.Random(77 + tpc * 10 + kc)
    for lf, lg, b, fs, gs in _cases(rng, [(2048, 2048, 64), (4096, 300, 33), (1024, 1024, 32)]):
        want = {p: O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in range(2)}
        for v in (1, 4):
            _check_batch(kmx, v, fs, gs, b, want)


def test_engines_agree_on_config2(kmx, env):
    rng = random.Random(2024)
    B, n = 64, 1024
    fs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    fd, gd = _dev_words(fs, 1, True), _dev_words(gs, 1, True)
    for v in (1, 2, 3, 4):
        outs = []
        for mode in ("0", "1"):
            env["KMX_TC"] = mode
            kb = kmx.KsBatch(v, B, n, n, 32, signed=True)
            h = kb(fd, gd)
            kb.status()
            outs.append(h.clone())
        assert torch.equal(outs[0], outs[1]), v
    got = _host_ints(outs[1], signed=True)
    assert got[5] == O.ks_mul_signed(1, fs[5], gs[5], 32, mode="native")


def test_all_ones_accumulators_past_2_31(kmx, env):
    # c4-sized ks4 operands (~34 KB): every accumulator column of the middle
    # tiles sums ~34K products of 255*255 > 2^31, read back as u32
    env.pop("KMX_TC", None)
    n, b = 4096, 128
    assert kmx.mul_engine(4, n, n, b) == "tensor"
    fs = [[(1 << b) - 1] * n]
    gs = [[(1 << b) - 1] * n]
    want = {0: O.ks_mul(1, fs[0], gs[0], b, mode="native")}
    for v in (1, 2, 3, 4):
        _check_batch(kmx, v, fs, gs, b, want)


def test_tc_peak_is_measured(kmx):
    peak = kmx.tc_peak(200)
    assert 1e14 < peak < 5e15


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_fused_pack_multiply(kmx, env, variant):
    # K1 fused into the tensor-core prologue (KMX_FUSE=1): operands packed in
    # shared memory, meta/prefix/range checks from the product's first CTA
    env.update(KMX_TC="1", KMX_FUSE="1")
    rng = random.Random(31 + variant)
    for lf, lg, b, fs, gs in _cases(rng, [(256, 256, 64), (1024, 1024, 64), (300, 77, 17), (5, 700, 96)]):
        want = {p: O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in range(2)}
        _check_batch(kmx, variant, fs, gs, b, want)
    B, n = 8, 1024
    fs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    gs = [[rng.randrange(-2**31, 2**31) for _ in range(n)] for _ in range(B)]
    want = {p: O.ks_mul_signed(1, fs[p], gs[p], 32, mode="native") for p in (0, 7)}
    _check_batch(kmx, variant, fs, gs, 32, want, signed=True)
    # a bad coefficient is still caught by the fused range check
    bad = [[0] * 16]
    bad[0][3] = 1 << 20
    with pytest.raises(ValueError):
        _check_batch(kmx, variant, bad, [[1] * 16], 16, {})
