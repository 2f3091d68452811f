"""GPU parity at the benchmarked batches: the exact inputs bench.py times
(bench.make_inputs, same seeds and batch sizes), so the kernel configuration
the bench measures -- the autotuned batch split and tensor-core tiling of that
(shape, batch) -- is the one checked.  Per config and variant:

  * the four variants are bit-identical on the whole batch;
  * a full-batch checksum: h(x0) == f(x0) g(x0) mod two primes for every pair
    (a size-independent property of the product);
  * the oracle (oracle/ks_oracle.py, Python ints) bit-exact on the first and
    last pair of every part a batch split or the host path's chunking makes;
  * the host-buffer path (kmx_ks_mul_host, pipelined chunks) equals the device
    path on the whole batch.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import bench  # noqa: E402

pytestmark = pytest.mark.gpu

PRIMES = ((1 << 31) - 1, 2147483629)
POINTS = (1234567, 987654321)


@pytest.fixture(scope="module")
def kmx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_0712_4046_b200 as k
    return k


def residues(words, p, signed=False):
    """[B, L, W] little-endian u32 words -> [B, L] int64 residues mod p."""
    w = np.ascontiguousarray(words).view(np.uint32).astype(np.int64)
    r = np.zeros(w.shape[:2], dtype=np.int64)
    base = 1
    for j in range(w.shape[2]):
        r = (r + (w[..., j] % p) * base) % p
        base = base * (1 << 32) % p
    if signed:  # two's complement: subtract 2^(32 W) where the top bit is set
        neg = (w[..., -1] >> 31) == 1
        r = np.where(neg, (r - base) % p, r)
    return r


def horner(res, x, p):
    acc = np.zeros(res.shape[0], dtype=np.int64)
    for i in range(res.shape[1] - 1, -1, -1):
        acc = (acc * x + res[:, i]) % p
    return acc


def checksum_ok(f, g, h, signed):
    for p, x in zip(PRIMES, POINTS):
        fe = horner(residues(f, p, signed), x, p)
        ge = horner(residues(g, p, signed), x, p)
        he = horner(residues(h, p, signed), x, p)
        if not np.all((fe * ge - he) % p == 0):
            return False
    return True


def run_variants(kmx, cfg, fh, gh):
    fd = torch.from_numpy(fh.view(np.int32)).cuda()
    gd = torch.from_numpy(gh.view(np.int32)).cuda()
    outs = {}
    for v in (1, 2, 3, 4):
        kb = kmx.KsBatch(v, cfg["batch"], cfg["n"], cfg["n"], cfg["b"], signed=cfg["signed"])
        out = kb.empty_out()
        kb(fd, gd, out)  # first call of the shape: schedule / tiling measured and cached
        kb.status()
        out.zero_()
        kb(fd, gd, out)  # the cached plan: what the bench's graph replays
        kb.status()
        outs[v] = out.cpu().numpy().view(np.uint32)
    return outs


def check_ks_config(kmx, cfg, pairs=None, host=True):
    fh, gh = bench.make_inputs(cfg)
    outs = run_variants(kmx, cfg, fh, gh)
    for v in (2, 3, 4):
        assert np.array_equal(outs[1], outs[v]), f"ks{v} differs from ks1 on the full batch"
    assert checksum_ok(fh, gh, outs[1], cfg["signed"]), "full-batch checksum"
    pairs = pairs if pairs is not None else bench.oracle_pairs(cfg, cfg["batch"])
    assert bench.check_pairs(cfg, 1, fh, gh, torch.from_numpy(outs[1].view(np.int32)), pairs)
    if host:
        fp = torch.from_numpy(fh.view(np.int32)).pin_memory().numpy().view(np.uint32)
        gp = torch.from_numpy(gh.view(np.int32)).pin_memory().numpy().view(np.uint32)
        for v in (1, 4):
            hp = kmx.ks_mul_host(v, fp, gp, cfg["b"], signed=cfg["signed"])
            assert np.array_equal(hp, outs[1]), f"host path ks{v}"


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_bench_config_full_batch(kmx, name):
    check_ks_config(kmx, bench.CONFIGS[name])


def test_bench_config3_full_batch(kmx):
    cfg = bench.CONFIGS["c3"]
    fh, gh = bench.make_inputs(cfg)
    fd, gd = torch.from_numpy(fh).cuda(), torch.from_numpy(gh).cuda()
    outs = {}
    for v in (1, 2, 3, 4):
        bb = kmx.BksBatch(v, cfg["batch"], cfg["lx"], cfg["ly"], cfg["b"])
        h = bb(fd, gd)
        bb.status()
        outs[v] = h.cpu().numpy()
    for v in (2, 3, 4):
        assert np.array_equal(outs[1], outs[v])
    # checksum: h(x0, y0) == f(x0, y0) g(x0, y0) mod p for all 256 pairs
    for p, (x, y) in zip(PRIMES, ((12345, 678), (99991, 31337))):
        def ev(a):
            a = np.asarray(a, dtype=np.int64) % p
            ys = horner(a.reshape(-1, a.shape[2]), y, p).reshape(a.shape[0], a.shape[1])
            return horner(ys, x, p)
        assert np.all((ev(fh) * ev(gh) - ev(outs[1])) % p == 0)
    assert bench.check_pairs(cfg, 4, fh, gh, torch.from_numpy(outs[4]), [0, 127, 128, 255])
    hp = kmx.bks_mul_host(4, fh, gh, cfg["b"])
    assert np.array_equal(hp, outs[4])


@pytest.mark.parametrize("n", [4096, 8192])
@pytest.mark.parametrize("b", [8, 32, 64, 128, 256])
def test_config5_large_bench_batch(kmx, n, b):
    # BASELINE config 5 large points at the batch the sweep times
    # (B = ceil(1e6 / (2n - 1)): 123 pairs at n=4096, 62 at n=8192)
    cfg = bench.c5_config(n, b)
    check_ks_config(kmx, cfg, pairs=[0, cfg["batch"] - 1], host=False)
