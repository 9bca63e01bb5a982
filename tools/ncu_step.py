"""Warm launches of the per-ply HBM-bound kernels of a config game (for ncu).

    python tools/ncu_step.py --game connect_four --batch 4194304

Runs 4 plies of lx_random_step, then 4 PGX plies (lx_sample + lx_env_step),
so `ncu -k regex:<kernel> -s 2 -c 1` captures a warm launch of each; prints
the batch, cubin key and state quads so tools/ncu_summary.py --step can turn
the captured DRAM bytes into bytes per env-ply.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_22609_b200 as lx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--game", default="connect_four")
p.add_argument("--batch", type=int, default=1 << 22)
a = p.parse_args()
g = lx.load_config_game(a.game)
st = g.init(batch_size=a.batch, seed=3)
for _ in range(4):
    g.random_step(st)
env = lx.LudaxEnvironment(g, auto_reset=True)
est = env.init(seed=2, batch_size=a.batch)
for _ in range(4):
    est = env.step_(est, env.random_actions(est))
torch.cuda.synchronize()
print(json.dumps({"game": a.game, "batch": a.batch, "cubin_key": g.lowered_key(),
                  "nq": g.info["nq"], "A": g.action_space_size}))
