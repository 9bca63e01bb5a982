"""Warm launches of the per-ply HBM-bound kernels of a config game (for ncu).

    python tools/ncu_step.py --game connect_four --batch 4194304

Runs 4 plies of lx_random_step, then a PGX env init + 4 plies with the
bool mask and an init + 4 plies with the bit-packed mask (lx_env_step with
the action sampled in the kernel), so `ncu -k regex:<kernel> -s S -c 1`
captures a warm launch of each (lx_random_step S=2, lx_env_step bool S=3,
lx_env_step bits S=8); prints
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
for fmt in ("bool", "bits"):
    env = lx.LudaxEnvironment(g, auto_reset=True, mask_format=fmt)
    est = env.init(seed=2, batch_size=a.batch)
    for _ in range(4):
        est = env.step_(est, env.RANDOM)
torch.cuda.synchronize()
print(json.dumps({"game": a.game, "batch": a.batch, "cubin_key": g.lowered_key(),
                  "nq": g.info["nq"], "A": g.action_space_size}))
