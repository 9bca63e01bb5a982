"""Warm launches of the interchange kernels (lx_export of every reference
field, lx_observe planes) of a config game at 2^20 envs, for ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_22609_b200 as lx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--game", default="connect_four")
p.add_argument("--batch", type=int, default=1 << 20)
a = p.parse_args()
g = lx.load_config_game(a.game)
final = lx.engine.playout_random(g, seed=3, batch_size=a.batch).final
for _ in range(3):
    g.export_device(final)
    g.observe_device(final, 0)
torch.cuda.synchronize()
print(a.game, a.batch, g.reference_state_bytes(), g.observation_planes * g.num_cells)
