"""bench.py's N>1 flow on CPU: torch.distributed.run launches two ranks of
`bench.py --stub` (gloo), which go through bench.run_distributed -- the same
code the GPU arm runs -- with each rank's episodes played by the oracle on
its own env shard.  The JSON line must equal one oracle run over the union
of the shards (weak scaling, no collective on the hot path)."""
import json
import os
import subprocess
import sys

import numpy as np

from conftest import ROOT
from oracle import oracle as O
from paper_2506_22609_b200 import rng


def _run(n, extra=()):
    port = 29700 + (os.getpid() % 200)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--stub",
           "--gpus", str(n), "--steps", "2", "--warmup", "3", "--batch", "96", *extra]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=240, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout          # rank 0 alone prints
    return json.loads(lines[0])


def test_two_rank_bench_flow_matches_one_run():
    line = _run(2)
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["scaling"] == "weak"
    assert line["config"]["global_batch"] == 192
    assert line["stub"] == {"rank0_extras": True, "ranks": 2}
    assert line["e2e"]["h2d_bytes_per_step"] == 96 * 8 * 2
    og = O.OracleGame("connect_four")
    want = np.zeros(6, np.int64)
    for e in (10_000, 10_001):
        st, steps = og.playout(state=og.init(192, seeds=rng.spawn_seeds(
            rng.episode_seed(0, 192, e), 192)))
        out = st["outcome"]
        want += [steps, (out == 1).sum(), (out == 2).sum(), (out == 0).sum(),
                 st["truncated"].sum(), 192]
    t = line["totals"]
    assert [t["env_steps"], t["p1_wins"], t["p2_wins"], t["draws"], t["truncated"],
            t["envs"]] == want.tolist()
    assert line["value"] == t["env_steps"] / (line["ms_per_step"] * 2 / 1000.0)


def test_reference_arm_rank0_only():
    line = _run(2, ("--impl", "reference", "--cpu-seconds", "0.2", "--no-extras"))
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
