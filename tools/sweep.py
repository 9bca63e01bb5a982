"""Batch-size sweep of the fused rollout for every config game (1 GPU).

    python tools/sweep.py [--games a,b] [--min-log2 10] [--max-log2 22]

Each point: 3 warm-up episodes, then episodes (seed hash_key(0, B, 10000+e))
timed with CUDA events until >= 0.25 s; batches up to 2^16 envs replay 20
captured episodes per CUDA-graph launch (they are launch-bound); prints one
JSON line per point.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_22609_b200 as lx  # noqa: E402
from paper_2506_22609_b200 import rng  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--games", default="tic_tac_toe,connect_four,hex,reversi,pente")
p.add_argument("--min-log2", type=int, default=10)
p.add_argument("--max-log2", type=int, default=22)
p.add_argument("--seconds", type=float, default=0.25)
a = p.parse_args()

for name in a.games.split(","):
    g = lx.load_config_game(name)
    for k in range(a.min_log2, a.max_log2 + 1):
        B = 1 << k
        out = g.empty_state(B)
        stats = torch.zeros(8, dtype=torch.int64, device="cuda")
        work = torch.zeros(16, dtype=torch.int64, device="cuda")
        acc = torch.zeros(8, dtype=torch.int64, device="cuda")

        def ep(e):
            g.rollout(seed=rng.episode_seed(0, B, e), out=out, batch_size=B, truncate=False,
                      check=False, stats=stats, work=work)
            acc.add_(stats)
        for e in range(3):
            ep(e)
        torch.cuda.synchronize()
        graph = None
        G = 20
        if B <= (1 << 16):          # launch-bound: replay G captured episodes per launch
            # each captured episode publishes its stats into its own row;
            # one sum per replay (no per-episode add kernel in the graph)
            per_ep = torch.zeros(G, 8, dtype=torch.int64, device="cuda")
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for e in range(G):
                    g.rollout(seed=rng.episode_seed(0, B, 10000 + e), out=out, batch_size=B,
                              truncate=False, check=False, stats=per_ep[e], work=work)
                acc.add_(per_ep.sum(0))
            graph.replay()
        torch.cuda.synchronize()
        acc.zero_()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n, ms = 0, 0.0
        while ms < a.seconds * 1000:
            reps = max(1, n)
            ev0.record()
            for e in range(reps):
                if graph is not None:
                    graph.replay()
                else:
                    ep(10000 + n + e)
            ev1.record()
            torch.cuda.synchronize()
            ms += ev0.elapsed_time(ev1)
            n += reps
        episodes = n * (G if graph is not None else 1)
        tot = acc.cpu().tolist()
        print(json.dumps({"game": name, "batch": B, "episodes": episodes,
                          "ms_per_episode": ms / episodes, "cuda_graph": graph is not None,
                          "env_steps_per_s": tot[0] / (ms / 1000),
                          "mean_plies": tot[0] / tot[5]}), flush=True)
