"""CPU stand-in for bench.py's GPU arm (test infrastructure only).

``python bench.py --stub`` runs bench.run_distributed -- warm-up, barriers,
timed episodes, max-over-ranks time, summed stats, the per-rank e2e leg,
rank-0 extras, the JSON line and teardown -- with each rank's episode played
by the CPU oracle on its own env shard and the collectives on gloo, so the
N>1 flow of the bench executes on a machine without GPUs
(tests/test_bench_dist.py launches it under torch.distributed.run).
"""

from __future__ import annotations

import contextlib
import time

import numpy as np
import torch
import torch.distributed as dist

import bench
from oracle import oracle as O
from paper_2506_22609_b200 import rng, shard


class StubArm:
    launches_per_episode = 0

    def __init__(self, args):
        self.args = args
        self.world_size, self.rank, self.local = bench.dist_env()
        if self.world_size > 1:
            dist.init_process_group("gloo")
        self.B = args.batch
        self.B_total = args.batch * self.world_size
        self.first, _ = shard.shard_range(self.rank, self.world_size, self.B)
        self.og = O.OracleGame(args.game)
        self.acc = np.zeros(8, np.int64)

    def _play(self, e):
        seeds = rng.spawn_seeds(rng.episode_seed(0, self.B_total, e), self.B, self.first)
        st, steps = self.og.playout(state=self.og.init(self.B, seeds=seeds),
                                    max_turns=self.args.max_turns)
        out = st["outcome"]
        return np.array([steps, (out == 1).sum(), (out == 2).sum(), (out == 0).sum(),
                         st["truncated"].sum(), self.B, 0, 0], np.int64)

    def episode(self, e):
        self.acc += self._play(e)

    def reset_totals(self):
        self.acc[:] = 0

    def barrier(self):
        if self.world_size > 1:
            dist.barrier()

    def sync(self):
        pass

    def clock_sampler(self):
        return contextlib.nullcontext(bench.ClockSampler(self.local, enabled=False))

    def timed(self, fn):
        t0 = time.perf_counter()
        fn()
        return 1000.0 * (time.perf_counter() - t0)

    def max_over_ranks(self, ms):
        t = torch.tensor([ms], dtype=torch.float64)
        shard.max_over_ranks(t)
        return float(t.item())

    def reduced_totals(self):
        t = torch.from_numpy(self.acc.copy())
        shard.reduce_stats(t)
        return t.tolist()

    def e2e(self):
        self.barrier()
        t0 = time.perf_counter()
        steps = int(self._play(20_000)[0])
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
        n = torch.tensor([steps], dtype=torch.int64)
        shard.max_over_ranks(t)
        shard.reduce_stats(n)
        self.barrier()
        return {"value": int(n.item()) / float(t.item()), "unit": bench.UNIT,
                "h2d_bytes_per_step": self.B * 8 * self.world_size,
                "d2h_bytes_per_step": self.B * self.world_size, "steps_timed": 1,
                "path": "stub (CPU oracle)"}

    def extras(self, value, ms_step, clock_mhz, totals):
        return {"stub": {"rank0_extras": True, "ranks": self.world_size}}

    def close(self):
        if self.world_size > 1:
            dist.destroy_process_group()
