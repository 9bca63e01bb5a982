"""lx_playout_host timing probe (1 GPU): streamed vs upload-first seeds, and
whether the driver exports the stream memory ops the streamed upload uses.

    python tools/probe_playout_host.py [--game connect_four] [--batch 4194304]
"""
import argparse
import ctypes
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
p.add_argument("--batch", type=int, default=1 << 22)
p.add_argument("--reps", type=int, default=10)
a = p.parse_args()
cu = ctypes.CDLL("libcuda.so.1")
print(json.dumps({"cuStreamWriteValue32_v2": hasattr(cu, "cuStreamWriteValue32_v2"),
                  "cuStreamWriteValue32": hasattr(cu, "cuStreamWriteValue32")}), flush=True)
g = lx.load_config_game(a.game)
B = a.batch
seeds = torch.from_numpy(rng.spawn_seeds(7, B).view(np.int64)).pin_memory()
outc = torch.empty(B, dtype=torch.int8).pin_memory()
stats = torch.zeros(8, dtype=torch.int64).pin_memory()
out = {}
for mode in ("streamed", "upload_first", "no_outcomes", "device_rollout"):
    def call():
        if mode == "device_rollout":
            g.rollout(batch_size=B, seed=7, store=False, check=False)
            torch.cuda.synchronize()
        else:
            g.playout_host(seeds=seeds, outcomes=outc if mode != "no_outcomes" else False,
                           stats=stats, upload_first=(mode == "upload_first"))
    for _ in range(3):
        call()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        call()
    out[mode] = (time.perf_counter() - t0) / a.reps * 1e3
print(json.dumps({"game": a.game, "batch": B, "ms_per_call": out}), flush=True)
