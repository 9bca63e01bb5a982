"""A/B timing of the per-ply kernels (lx_random_step, lx_env_step with the
action sampled in the kernel, bool / bit masks) under lowering variants
chosen by env overrides, e.g.

    python tools/ab_envstep.py --game connect_four --variant "" --variant LX_STEP_MINB=4
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
p.add_argument("--plies", type=int, default=64)
p.add_argument("--variant", action="append", default=[])
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
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    out = {"env": env}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = g.init(B, seed=1)
    for _ in range(4):
        g.random_step(st)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(a.plies):
        g.random_step(st)
    ev1.record()
    torch.cuda.synchronize()
    out["random_step_G"] = B / (ev0.elapsed_time(ev1) / a.plies / 1e3) / 1e9
    for fmt in ("bool", "bits"):
        e = lx.LudaxEnvironment(g, auto_reset=True, mask_format=fmt)
        s = e.init(seed=2, batch_size=B)
        for _ in range(8):
            s = e.step_(s, e.RANDOM)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(a.plies):
            s = e.step_(s, e.RANDOM)
        ev1.record()
        torch.cuda.synchronize()
        out[f"env_{fmt}_G"] = B / (ev0.elapsed_time(ev1) / a.plies / 1e3) / 1e9
        out[f"digest_{fmt}"] = s.game_state.digest() if B <= (1 << 20) else None
        # checksum of the last ply's mask (equal across variants = same masks)
        m = s.mask_bool()
        if m is not None:
            mi = m.to(torch.int64).reshape(B, -1)
            w = torch.arange(1, mi.shape[1] + 1, device=mi.device, dtype=torch.int64)
            out[f"mask_sum_{fmt}"] = int((mi * w).sum().item() +
                                         (mi.sum(1) * torch.arange(B, device=mi.device)).sum().item())
    res["variants"].append(out)
print(json.dumps(res))
