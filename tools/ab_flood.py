"""A/B timing of the fused rollout with the warp-cooperative reach-set flood
(default lowering) vs the per-lane flood (LX_COOP_FLOOD=0), same seeds.

    python tools/ab_flood.py --game hex --batch 4194304
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
p.add_argument("--game", default="hex")
p.add_argument("--batch", type=int, default=1 << 22)
p.add_argument("--reps", type=int, default=10)
a = p.parse_args()
with open(os.path.join(lx.game.GAMES_DIR, f"{a.game}.ldx")) as f:
    text = f.read()
games = {"coop": lx.load_game(text)}
os.environ["LX_COOP_FLOOD"] = "0"
games["solo"] = lx.load_game(text)
B = a.batch
res = {"game": a.game, "batch": B}
for name, g in games.items():
    out = g.empty_state(B)
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    for e in range(3):
        g.rollout(seed=rng.episode_seed(0, B, e), out=out, batch_size=B, truncate=False,
                  check=False, stats=stats)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(a.reps)]
    e0.record()
    for e in range(a.reps):         # lx_rollout overwrites its stats vector
        g.rollout(seed=rng.episode_seed(0, B, 10000 + e), out=out, batch_size=B, truncate=False,
                  check=False, stats=per[e])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    stats = sum(per)
    steps = int(stats[0].item())
    res[name] = {"key": g.lowered_key(), "ms_per_episode": ms / a.reps,
                 "env_steps_per_s": steps / (ms / 1e3), "stats": stats.cpu().tolist()}
res["speedup"] = res["coop"]["env_steps_per_s"] / res["solo"]["env_steps_per_s"]
res["same_stats"] = res["coop"]["stats"] == res["solo"]["stats"]
print(json.dumps(res))
