"""The N>1 bench path on CPU: two gloo ranks, each multiplying its own
(independent) batch; timings are combined as the max over ranks and the
products counted over the whole job (weak scaling, no data-path collective)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = bench.rank_env()
    assert (r, w, lr) == (rank, world, rank)
    # each rank draws its own seeded inputs (independent pairs)
    f0, _ = bench.make_inputs(bench.CONFIGS["c1"], rank)
    local_ms = 10.0 * (rank + 1)
    t = bench.max_over_ranks(local_ms, dist, torch.device("cpu"))
    # every rank also checks its shard differs from rank 0's
    flat = torch.from_numpy(f0[:1].astype("int64").reshape(-1))
    gathered = [torch.zeros_like(flat) for _ in range(world)]
    dist.all_gather(gathered, flat)
    distinct = not torch.equal(gathered[0], gathered[1])
    q.put((rank, t, bench.job_products(64, w), distinct))
    dist.destroy_process_group()


def test_two_rank_timing_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [20.0, 20.0]   # max over ranks
    assert all(r[2] == 128 for r in res)         # weak scaling: products of the whole job
    assert all(r[3] for r in res)                # independent inputs per rank
