"""One warm-up + one measured fused rollout of a config game (for ncu).

    python tools/ncu_rollout.py --game connect_four --batch 1048576
Prints the env steps of the measured (2nd) lx_rollout launch so ncu
instruction counts can be normalised per env step.
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
p.add_argument("--game", default="connect_four")
p.add_argument("--batch", type=int, default=1 << 20)
a = p.parse_args()
g = lx.load_config_game(a.game)
out = g.empty_state(a.batch)
for e in (0, 10000):
    _, stats = g.rollout(seed=rng.episode_seed(0, a.batch, e), out=out, batch_size=a.batch,
                         truncate=False, check=False)
torch.cuda.synchronize()
s = stats.cpu().tolist()
print(json.dumps({"game": a.game, "batch": a.batch, "cubin_key": g.lowered_key(),
                  "env_steps": s[0], "envs": s[5], "nq": g.info["nq"],
                  "rollout_blocks": g.native.info.rollout_blocks}))
