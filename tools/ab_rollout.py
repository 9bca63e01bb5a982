"""A/B timing of the fused rollout of one game (store vs outcomes-only).

    LX_CONN_UF=0 python tools/ab_rollout.py --game hex --batch 4194304
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
p.add_argument("--reps", type=int, default=5)
a = p.parse_args()
g = lx.load_config_game(a.game)
B = a.batch
out = g.empty_state(B)
stats = torch.zeros(8, dtype=torch.int64, device="cuda")
outc = torch.empty(B, dtype=torch.int8, device="cuda")
res = {"game": a.game, "batch": B, "conn_uf": os.environ.get("LX_CONN_UF", "1")}
for store in (True, False):
    for e in range(2):
        g.rollout(seed=rng.episode_seed(0, B, e), out=out, batch_size=B, truncate=False,
                  check=False, stats=stats, store=store, outcomes=None if store else outc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 0
    e0.record()
    for e in range(a.reps):
        g.rollout(seed=rng.episode_seed(0, B, 10000 + e), out=out, batch_size=B, truncate=False,
                  check=False, stats=stats, store=store, outcomes=None if store else outc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    res["store" if store else "outcomes_only"] = {"ms": ms, "G_steps_s": int(stats[0]) / ms / 1e6}
print(json.dumps(res))
