"""A/B timing of the fused rollout under lowering variants chosen by env
overrides (same seeds, stats compared), e.g.

    python tools/ab_env.py --game connect_four --variant LX_ROLLOUT_MINB=2 \
        --variant LX_ROLLOUT_MINB=3
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
p.add_argument("--batch", type=int, default=1 << 22)
p.add_argument("--reps", type=int, default=10)
p.add_argument("--variant", action="append", default=[],
               help="comma-separated K=V env overrides; '' = default lowering")
a = p.parse_args()
with open(os.path.join(lx.game.GAMES_DIR, f"{a.game}.ldx")) as f:
    text = f.read()
B = a.batch
res = {"game": a.game, "batch": B, "variants": []}
for var in (a.variant or [""]):
    env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    g = lx.load_game(text)
    g.lowered_key()
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    out = g.empty_state(B)
    for e in range(3):
        g.rollout(seed=rng.episode_seed(0, B, e), out=out, batch_size=B, truncate=False,
                  check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outs = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(a.reps)]
    e0.record()
    for e in range(a.reps):
        g.rollout(seed=rng.episode_seed(0, B, 10000 + e), out=out, batch_size=B,
                  truncate=False, check=False, stats=outs[e])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    steps = sum(int(s[0].item()) for s in outs)
    res["variants"].append({"env": env, "key": g.lowered_key(), "ms_per_episode": ms / a.reps,
                            "env_steps_per_s": steps / (ms / 1e3),
                            "stats0": outs[0].cpu().tolist()})
v = res["variants"]
res["same_stats"] = all(x["stats0"] == v[0]["stats0"] for x in v)
print(json.dumps(res))
