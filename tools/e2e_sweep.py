"""End-to-end env steps/s vs batch size through the C-ABI host-buffer calls
(lx_playout_host_async / _wait, two episodes in flight, pinned host seeds in,
host outcomes + stats out), beside the device-timed fused rollout of the same
batch (1 GPU).

    python tools/e2e_sweep.py [--game connect_four] [--min-log2 10] [--max-log2 22]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_22609_b200 as lx  # noqa: E402
from paper_2506_22609_b200 import rng  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--game", default="connect_four")
p.add_argument("--min-log2", type=int, default=10)
p.add_argument("--max-log2", type=int, default=22)
p.add_argument("--seconds", type=float, default=0.3)
a = p.parse_args()
g = lx.load_config_game(a.game)
for k in range(a.min_log2, a.max_log2 + 1):
    B = 1 << k
    n_buf = 6
    seeds = [torch.from_numpy(rng.spawn_seeds(rng.episode_seed(0, B, 40000 + e), B)
                              .view(np.int64)).pin_memory() for e in range(n_buf)]
    outc = [torch.empty(B, dtype=torch.int8).pin_memory() for _ in range(n_buf)]
    stats = [torch.zeros(8, dtype=torch.int64).pin_memory() for _ in range(n_buf)]

    def run(n):
        pending, steps = [], 0
        for it in range(n):
            j = it % n_buf
            pending.append((j, g.playout_host_async(seeds=seeds[j], outcomes=outc[j],
                                                    stats=stats[j])))
            if len(pending) > 2:
                jj, t = pending.pop(0)
                g.playout_host_wait(t)
                steps += int(stats[jj][0])
        for jj, t in pending:
            g.playout_host_wait(t)
            steps += int(stats[jj][0])
        return steps
    run(4)
    n = 4
    while True:
        t0 = time.perf_counter()
        steps = run(n)
        dt = time.perf_counter() - t0
        if dt >= a.seconds or n >= 4096:
            break
        n *= 2
    # device-timed fused rollout of the same batch (seeds spawned on the device)
    out = g.empty_state(B)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.zeros(8, dtype=torch.int64, device="cuda")
    g.rollout(seed=rng.episode_seed(0, B, 1), out=out, batch_size=B, stats=st, check=False)
    torch.cuda.synchronize()
    ev0.record()
    dsteps = 0
    reps = max(1, min(n, 64))
    accs = []
    for e in range(reps):
        s_e = torch.zeros(8, dtype=torch.int64, device="cuda")
        g.rollout(seed=rng.episode_seed(0, B, 40000 + e), out=out, batch_size=B, stats=s_e,
                  check=False)
        accs.append(s_e)
    ev1.record()
    torch.cuda.synchronize()
    dsteps = sum(int(x[0]) for x in accs)
    print(json.dumps({"game": a.game, "batch": B, "episodes": n,
                      "e2e_env_steps_per_s": steps / dt,
                      "us_per_episode_e2e": dt / n * 1e6,
                      "device_env_steps_per_s": dsteps / (ev0.elapsed_time(ev1) / 1e3),
                      "h2d_bytes_per_episode": 8 * B, "d2h_bytes_per_episode": B + 64}),
          flush=True)
