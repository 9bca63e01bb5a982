"""Every-env oracle parity of a full 2^22-env benchmark episode (1 GPU).

bench.py checks every env of the benchmarked episode for TTT and C4 and the
first 2^20 envs for Hex, Reversi and Pente (their oracle replays take
minutes); this tool checks all 2^22 for the games given, with the same
episode seed (the bench's last timed episode, 10019) and the same checker
(bench.parity_check: every reference GameState field of every env).

    python tools/full_parity.py [--games hex,reversi,pente] [--batch 4194304]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_22609_b200 as lx  # noqa: E402
from paper_2506_22609_b200 import rng  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--games", default="hex,reversi,pente")
p.add_argument("--batch", type=int, default=1 << 22)
p.add_argument("--episode", type=int, default=10019)
a = p.parse_args()
B = a.batch
for name in a.games.split(","):
    g = lx.load_config_game(name)
    state = g.empty_state(B)
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    work = torch.zeros(16, dtype=torch.int64, device="cuda")
    t0 = time.perf_counter()
    bench.native_rollout(g, state, B, 200, rng.episode_seed(0, B, a.episode), 0, stats, work)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    par, cpu = bench.parity_check(name, g, state, B, a.episode, B, 200)
    print(json.dumps({"game": name, "batch": B, "episode": a.episode,
                      "device_env_steps": int(stats[0].item()), "device_wall_s": dev_s,
                      "parity": par, "oracle": cpu}), flush=True)
    del state
    torch.cuda.empty_cache()
