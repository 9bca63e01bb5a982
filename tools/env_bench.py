"""PGX-style env-step throughput (LudaxEnvironment.step_ on device).

    python tools/env_bench.py [--batch 1048576] [--plies 64]

Per ply: lx_sample (uniform legal action per env, reads the state) then
lx_env_step (apply, rewards, flags, next legal mask).  Reports env steps/s
and the HBM bandwidth each kernel achieves against its algorithmic bytes.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_22609_b200 as lx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--games", default="tic_tac_toe,connect_four,hex,reversi,pente")
p.add_argument("--batch", type=int, default=1 << 20)
p.add_argument("--plies", type=int, default=64)
a = p.parse_args()
peak = 6366.5
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as f:
        peak = json.load(f)["hbm_gbs"]
except Exception:
    pass
for name in a.games.split(","):
    env = lx.LudaxEnvironment(name, auto_reset=True)
    B = a.batch
    st = env.init(seed=1, batch_size=B)
    acts = env.random_actions(st)
    for _ in range(3):
        acts = env.random_actions(st)
        st = env.step_(st, acts)
    torch.cuda.synchronize()
    # events back to back, one synchronize at the end (a per-ply synchronize
    # would put the host's launch latency on an idle GPU into each interval)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.plies + 1)]
    e[0].record()
    for p in range(a.plies):
        acts = env.random_actions(st)
        e[2 * p + 1].record()
        st = env.step_(st, acts)
        e[2 * p + 2].record()
    torch.cuda.synchronize()
    t_sample = sum(e[2 * p].elapsed_time(e[2 * p + 1]) for p in range(a.plies))
    t_step = sum(e[2 * p + 1].elapsed_time(e[2 * p + 2]) for p in range(a.plies))
    nq, A = env.game.info["nq"], env.num_actions
    b_sample = B * (nq * 16 + 8)
    b_step = B * (2 * nq * 16 + 8 + A + 8 + 6)
    ms_s, ms_t = t_sample / a.plies, t_step / a.plies
    print(json.dumps({
        "game": name, "batch": B, "env_steps_per_s": B / ((ms_s + ms_t) / 1e3),
        "sample": {"ms": ms_s, "GBps": b_sample / ms_s / 1e6, "frac": b_sample / ms_s / 1e6 / peak},
        "env_step": {"ms": ms_t, "GBps": b_step / ms_t / 1e6, "frac": b_step / ms_t / 1e6 / peak,
                     "bytes_per_env": b_step / B}}), flush=True)
