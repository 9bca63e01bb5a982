"""Small-batch latency of the fused rollout (1 GPU): ms per episode at a
fixed batch as the ply cap grows, so the fixed cost of a launch (claim,
init, store, stats publish) separates from the per-ply critical path.

    python tools/latency_probe.py [--game tic_tac_toe] [--batch 1024] [--caps 0,1,2,...]

Every point replays 20 captured episodes per CUDA-graph launch (as bench.py's
per-config block does for batches <= 2^16) and prints one JSON line.
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
p.add_argument("--game", default="tic_tac_toe")
p.add_argument("--batch", type=int, default=1024)
p.add_argument("--caps", default="0,1,2,3,4,5,6,7,8,9,200")
p.add_argument("--reps", type=int, default=200)
p.add_argument("--variant", default="",
               help="comma-separated K=V lowering env overrides (tools/ab_env.py style)")
a = p.parse_args()

env = dict(kv.split("=", 1) for kv in a.variant.split(",") if kv)
os.environ.update(env)
with open(os.path.join(lx.game.GAMES_DIR, f"{a.game}.ldx")) as f:
    g = lx.load_game(f.read())
g.lowered_key()
B = a.batch
out = g.empty_state(B)
work = torch.zeros(16, dtype=torch.int64, device="cuda")
G = 20
# reference point: a graph of G trivial kernels (the per-node launch floor)
z = torch.zeros(G, 8, dtype=torch.int64, device="cuda")
gz = torch.cuda.CUDAGraph()
with torch.cuda.graph(gz):
    for e in range(G):
        z[e].zero_()
# >= 200 ms of replays first: the SM clock must be up before any timing
import time  # noqa: E402
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.2:
    gz.replay()
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    gz.replay()
e1.record()
torch.cuda.synchronize()
print(json.dumps({"trivial_kernel_node_us": e0.elapsed_time(e1) / (a.reps * G) * 1e3}), flush=True)
for cap in [int(c) for c in a.caps.split(",")]:
    per_ep = torch.zeros(G, 8, dtype=torch.int64, device="cuda")
    for e in range(3):
        g.rollout(seed=rng.episode_seed(0, B, e), out=out, batch_size=B, max_turns=cap,
                  truncate=False, check=False, stats=per_ep[0], work=work)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for e in range(G):
            g.rollout(seed=rng.episode_seed(0, B, 10000 + e), out=out, batch_size=B,
                      max_turns=cap, truncate=False, check=False, stats=per_ep[e], work=work)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.05:
        graph.replay()
        torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(a.reps):
        graph.replay()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / (a.reps * G)
    tot = per_ep.sum(0).tolist()
    print(json.dumps({"game": a.game, "batch": B, "variant": env, "max_turns": cap, "us_per_episode": ms * 1e3,
                      "env_steps_per_episode": tot[0] / G,
                      "env_steps_per_s": tot[0] / G / (ms / 1e3)}), flush=True)
