"""Host RNG vs the reference's vectors; env sharding over gloo ranks."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_22609_b200 import rng, shard


def test_host_rng_matches_reference(golden_meta):
    r = golden_meta["kat"]["rng"]
    seeds = rng.spawn_seeds(12345, 16)
    assert [str(int(x)) for x in seeds] == r["spawn_12345_16"]
    u = rng.uniform(seeds, np.arange(16, dtype=np.uint64) * 7)
    assert [float.hex(float(x)) for x in u] == r["uniform_hex"]
    for key, v in r["episode_keys"].items():
        b, e = map(int, key.split("_"))
        assert str(rng.episode_seed(0, b, e)) == v


def test_split_even_covers():
    for total in (1, 7, 1000):
        for ws in (1, 2, 3, 8):
            spans = [shard.split_even(total, ws, r) for r in range(ws)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import oracle as O
    B = 512
    first, last = shard.shard_range(rank, ws, B)
    og = O.OracleGame("connect_four")
    st, steps = og.playout(state=og.init(B, seeds=rng.spawn_seeds(99, B, first=first)))
    stats = torch.tensor([steps, (st["outcome"] == 1).sum(), (st["outcome"] == 2).sum(),
                          (st["outcome"] == 0).sum(), st["truncated"].sum(), B],
                         dtype=torch.int64)
    shard.reduce_stats(stats)
    t = torch.tensor([float(rank)])
    shard.max_over_ranks(t)
    if rank == 0:
        out.put((stats.tolist(), float(t)))
    dist.destroy_process_group()


def test_two_rank_gloo_shards_equal_one_run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    stats, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    from oracle import oracle as O
    og = O.OracleGame("connect_four")
    st, steps = og.playout(state=og.init(1024, seeds=rng.spawn_seeds(99, 1024)))
    assert stats == [steps, int((st["outcome"] == 1).sum()), int((st["outcome"] == 2).sum()),
                     int((st["outcome"] == 0).sum()), int(st["truncated"].sum()), 1024]
    assert tmax == 1.0
