"""Benchmark: env steps/s of uniform-random rollouts, every BASELINE config.

Metric and protocol follow the reference benchmark (reference:
pkg/src/boardlang/evaluation.py:197-233): one step of this bench = one
synchronized batch episode -- B envs started from the program's start
position with per-env seeds spawn(hash_key(0, B_total, e), global index),
played with uniform legal actions until every env has terminated (cap 200
plies); env steps = live envs advanced by one ply, summed.

The headline line is configs[1] (Connect Four, 2^22 envs per GPU).  At N=1
the line also carries ``per_config``: every BASELINE.json config measured in
the same run -- Tic-Tac-Toe at B=1024 (configs[0], the reference's CPU-sized
case) and at 2^22, Connect Four, Hex, Reversi and Pente at 2^22 -- each with
its own timed episodes, roofline, e2e legs, CPU baseline and an oracle
parity check of the benchmarked episode's final states.

``e2e`` goes through the reference-facing C-ABI with host buffers
(lx_playout_host_async / _wait: pinned host seeds in, host outcomes + stats
out, every copy inside the timed region); ``e2e_python`` is the same metric
through the Python B200Game.rollout API with torch-managed copies.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--game G]
  python bench.py --impl reference ...      # CPU reference arm (oracle port)

Under torchrun each rank plays its own slice [rank*B, (rank+1)*B) of the
global env index space (weak scaling, no collective on the hot path); one
all-reduce (MAX) of the device time and one (SUM) of the stats after the
timed region.  ``run_distributed`` holds that flow; the GPU arm and the CPU
test stub (tests/test_bench_dist.py, gloo world size 2) both run through it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env steps/sec (uniform-random rollouts) vs batch size at 1/2/4/8 B200"
UNIT = "env_steps/s"
GAME_FILES = {"connect_four": "Connect Four 6x7", "tic_tac_toe": "Tic-Tac-Toe",
              "hex": "Hex 11x11", "reversi": "Reversi 8x8", "pente": "Pente 19x19",
              "gomoku": "Gomoku 15x15", "yavalath": "Yavalath (hexagon 9)",
              "english_draughts": "English Draughts 8x8",
              "dai_hasami_shogi": "Dai Hasami Shogi 9x9", "wolf_and_sheep": "Wolf and Sheep 8x8",
              "gridworld": "Frozen Lake gridworld 4x4"}

# BASELINE.json configs measured at N=1: (label, game, batch, timed steps,
# envs of the benchmarked episode replayed by the oracle).  The parity sample
# is every env where the oracle finishes in seconds on the box's host cores
# (TTT, C4), else a 2^20 prefix of the same episode.
GRAPH_MAX_BATCH = 1 << 16        # per-config episodes this small are replayed from a CUDA graph
PER_CONFIG = (
    ("configs[0]", "tic_tac_toe", 1024, 400, 1024),
    ("configs[0]@2^22", "tic_tac_toe", 1 << 22, 20, 1 << 22),
    ("configs[1]", "connect_four", 1 << 22, 20, 1 << 22),
    ("configs[2]", "hex", 1 << 22, 20, 1 << 20),
    ("configs[3]", "reversi", 1 << 22, 20, 1 << 20),
    ("configs[4]", "pente", 1 << 22, 20, 1 << 20),
)


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=400)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--batch", type=int, default=1 << 22, help="envs per GPU")
    p.add_argument("--game", default="connect_four", choices=sorted(GAME_FILES))
    p.add_argument("--max-turns", type=int, default=200)
    p.add_argument("--impl", default="b200", choices=("b200", "reference"))
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="target CPU time of the bounded CPU-baseline sample")
    p.add_argument("--no-extras", action="store_true",
                   help="skip the e2e / step-kernel / cpu-baseline / per-config legs")
    p.add_argument("--no-per-config", action="store_true",
                   help="headline config only (skip the per_config block)")
    p.add_argument("--parity-scale", type=float, default=1.0,
                   help="scale the per-config oracle parity samples (quick runs)")
    p.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)   # CPU test arm
    return p.parse_args(argv)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, enabled=True):
        self.index = index
        self.rows = []
        self._proc = None
        self.enabled = enabled

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)          # first sample lands before the timed region
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *exc):
        if self._proc is None:
            return
        time.sleep(0.06)
        self._proc.terminate()
        try:
            out, _ = self._proc.communicate(timeout=5)
        except Exception:
            self._proc.kill()
            out = ""
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU arm
def cpu_model():
    """Host CPU model name (BASELINE.md section 2 asks for it beside core counts)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_rate(game, batch_total, seconds, threads, max_turns):
    """Oracle port (plain C, all host threads) on a bounded sample of the same
    workload: the first envs of episode 10000, repeated until ~seconds."""
    from oracle import oracle as O
    og = O.OracleGame(game)
    seed = O.hash_key3(0, batch_total, 10000)
    n = 4096
    steps_total, t_total = 0, 0.0
    while t_total < seconds:
        seeds = O.spawn_seeds(seed, n)
        st = og.init(n, seeds=seeds)
        t0 = time.perf_counter()
        _, steps = og.playout(state=st, max_turns=max_turns, threads=threads)
        dt = time.perf_counter() - t0
        steps_total += steps
        t_total += dt
        if dt < seconds / 8:
            n = min(n * 2, batch_total)
    return steps_total / t_total, steps_total, t_total, n


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    B_total = args.batch * max(ws, args.gpus)
    rates = []
    per = max(args.cpu_seconds / max(args.steps, 1), 0.02)
    for w in range(args.warmup):
        cpu_rate(args.game, B_total, min(per, 1.0), threads, args.max_turns)
    sample = None
    for _ in range(args.steps):
        r, steps, dt, n = cpu_rate(args.game, B_total, per, threads, args.max_turns)
        rates.append(r)
        sample = f"{steps} env steps of the first {n} envs of episode 10000, {dt:.1f}s"
    value = statistics.mean(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * per, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config(args, ws),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if not args.no_extras:
        line["reference_numpy"] = numpy_reference_rate(args.game, seconds=3.0,
                                                       max_turns=args.max_turns)
        line["reference_numpy_all_cores"] = numpy_reference_mp(args.game, seconds=6.0,
                                                               max_turns=args.max_turns)
    print(json.dumps(line), flush=True)


def _ref_dir():
    return os.path.join(ROOT, "baseline", "_ref")


def _mp_worker(args):
    """One forked worker of numpy_reference_mp: the unmodified reference
    _run_episode on its own episodes until `seconds` of loop time."""
    game, wid, seconds, max_turns, batch = args
    os.environ["OMP_NUM_THREADS"] = "1"
    sys.path.insert(0, _ref_dir())
    import numpy as np
    import boardlang
    from boardlang import evaluation, rng as rrng
    with open(os.path.join(ROOT, "paper_2506_22609_b200", "games", f"{game}.ldx")) as f:
        g = boardlang.load_game(f.read())
    steps, t, e = 0, 0.0, 0
    while t < seconds:
        seed = rrng.hash_key(np.uint64(0), np.uint64(batch), np.uint64(10_000 + 1000 * wid + e))
        s, dt = evaluation._run_episode(g, batch, seed, max_turns)
        steps += s
        t += dt
        e += 1
    return steps, t, e


def numpy_reference_mp(game, seconds, max_turns, batch=1024):
    """The unmodified reference on every host core:
    os.cpu_count() forked workers, OMP_NUM_THREADS=1, each timing its own
    _run_episode loop (evaluation.py:197-211) on independent B=1024 episodes;
    rate = sum of steps / max worker loop time.  Context only."""
    if not os.path.isdir(os.path.join(_ref_dir(), "boardlang")):
        return {"error": "baseline/_ref is not staged (build() installs it from /root/reference)"}
    try:
        import multiprocessing as mp
        n = os.cpu_count() or 1
        with mp.get_context("fork").Pool(n) as pool:
            res = pool.map(_mp_worker, [(game, w, seconds, max_turns, batch) for w in range(n)])
        steps = sum(r[0] for r in res)
        tmax = max(r[1] for r in res)
        return {"value": steps / tmax, "unit": UNIT, "cores": n, "kind": "reference",
                "sample": f"{sum(r[2] for r in res)} episodes x {batch} envs, {n} forked "
                          f"workers of boardlang.evaluation._run_episode, ~{seconds:.0f}s each"}
    except Exception as exc:
        return {"error": repr(exc)[:200]}


def numpy_reference_rate(game, seconds, max_turns, batch=1024):
    """For context only: the unmodified reference (pip-installed into
    baseline/_ref) timed through its own _run_episode (evaluation.py:197-211),
    one process, B=1024, on the same game program."""
    ref_dir = _ref_dir()
    if not os.path.isdir(os.path.join(ref_dir, "boardlang")):
        return {"error": "baseline/_ref is not staged (build() installs it from /root/reference)"}
    try:
        sys.path.insert(0, ref_dir)
        import numpy as np
        import boardlang
        from boardlang import evaluation, rng as rrng
        with open(os.path.join(ROOT, "paper_2506_22609_b200", "games", f"{game}.ldx")) as f:
            g = boardlang.load_game(f.read())
        steps, t, e = 0, 0.0, 0
        while t < seconds:
            seed = rrng.hash_key(np.uint64(0), np.uint64(batch), np.uint64(10_000 + e))
            s, dt = evaluation._run_episode(g, batch, seed, max_turns)
            steps += s
            t += dt
            e += 1
        return {"value": steps / t, "unit": UNIT, "cores": 1, "episodes": e,
                "sample": f"{e} episodes x {batch} envs via boardlang.evaluation._run_episode"}
    except Exception as exc:              # context only; never fail the bench
        return {"error": repr(exc)[:200]}
    finally:
        if ref_dir in sys.path:
            sys.path.remove(ref_dir)


def config(args, ws, game=None, batch=None):
    game = game or args.game
    batch = batch or args.batch
    return {"workload": f"{GAME_FILES[game]} uniform-random rollouts, "
                        f"{batch} envs per GPU, full episodes (cap {args.max_turns} plies)",
            "game": game, "batch_per_gpu": batch,
            "global_batch": batch * ws, "max_turns": args.max_turns,
            "parallelism": f"env-shard x{ws}",
            "l2": "final states written each step (32-128 B/env: > 126 MB L2 at 2^22 envs); "
                  "the rollout reads no input but its seeds, so there is nothing to flush"}


# ------------------------------------------------------------------ shared distributed flow
def run_distributed(args, arm):
    """Warm-up, barrier, K timed episodes, max-over-ranks time, summed stats,
    e2e leg on every rank, rank-0 extras, one JSON line from rank 0.  `arm`
    is the GPU arm (below) or the CPU stub of tests/test_bench_dist.py."""
    ws, rank = arm.world_size, arm.rank
    for w in range(args.warmup):
        arm.episode(w)
    arm.reset_totals()
    arm.barrier()
    arm.sync()
    with arm.clock_sampler() as clk:
        ms = arm.timed(lambda: [arm.episode(10_000 + e) for e in range(args.steps)])
    ms_max = arm.max_over_ranks(ms)
    tot = arm.reduced_totals()
    arm.barrier()
    value = tot[0] / (ms_max / 1000.0)
    extras = {}
    if not args.no_extras:
        # e2e: the reference-facing C-ABI with host buffers (lx_playout_host_async
        # / _wait); e2e_python: the Python B200Game.rollout pipeline beside it
        if hasattr(arm, "e2e_host"):
            extras["e2e"] = arm.e2e_host()
            extras["e2e_python"] = arm.e2e()
        else:
            extras["e2e"] = arm.e2e()
    if rank == 0 and not args.no_extras:
        extras.update(arm.extras(value, ms_max / args.steps, clk.summary().get("sm_mhz"), tot))
        if hasattr(arm, "e2e_host"):
            for k in ("e2e", "e2e_python"):
                rl = e2e_roofline(extras.get(k), tot[0] / args.steps, value, ws)
                if rl:
                    extras[k]["roofline"] = rl
    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic (seeded random play from the start position)",
                "config": config(args, ws), "clocks": clk.summary(),
                "gpu_launches": args.steps * arm.launches_per_episode,
                "totals": {"env_steps": tot[0], "p1_wins": tot[1], "p2_wins": tot[2],
                           "draws": tot[3], "truncated": tot[4], "envs": tot[5]},
                "mean_plies": tot[0] / max(tot[5], 1)}
        line.update(extras)
        print(json.dumps(line), flush=True)
    arm.barrier()
    arm.close()
    return line


# ------------------------------------------------------------------ GPU arm
class GpuArm:
    launches_per_episode = 1           # one lx_rollout per episode

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        import paper_2506_22609_b200 as lx
        from paper_2506_22609_b200 import rng, shard
        self.torch, self.dist, self.lx, self.rng, self.shard = torch, dist, lx, rng, shard
        self.args = args
        self.world_size, self.rank, self.local = dist_env()
        torch.cuda.set_device(self.local)
        if self.world_size > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.game = lx.load_config_game(args.game)
        self.B = args.batch
        self.B_total = args.batch * self.world_size
        self.first, _ = shard.shard_range(self.rank, self.world_size, self.B)
        self.state = self.game.empty_state(self.B)
        self.stats = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.work = torch.zeros(16, dtype=torch.int64, device="cuda")
        self.acc = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.last_episode = None

    # -- flow hooks --
    def episode(self, e):
        seed = self.rng.episode_seed(0, self.B_total, e)
        native_rollout(self.game, self.state, self.B, self.args.max_turns, seed, self.first,
                       self.stats, self.work)
        self.acc.add_(self.stats)
        self.last_episode = e

    def reset_totals(self):
        self.torch.cuda.synchronize()
        self.acc.zero_()

    def barrier(self):
        if self.world_size > 1:
            self.dist.barrier()

    def sync(self):
        self.torch.cuda.synchronize()

    def clock_sampler(self):
        return ClockSampler(self.local)

    def timed(self, fn):
        torch = self.torch
        stream = torch.cuda.current_stream()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1)

    def max_over_ranks(self, ms):
        t = self.torch.tensor([ms], dtype=self.torch.float64, device="cuda")
        self.shard.max_over_ranks(t)
        return float(t.item())

    def reduced_totals(self):
        tot = self.acc.clone()
        self.shard.reduce_stats(tot)
        return tot.cpu().tolist()

    def e2e(self):
        return measure_e2e(self.args, self.game, self.rng, self.B, self.B_total, self.first,
                           self.world_size)

    def e2e_host(self):
        return measure_e2e_host(self.args, self.game, self.rng, self.B, self.B_total, self.first,
                                self.world_size)

    def extras(self, value, ms_step, clock_mhz, totals):
        out = measure_extras(self.args, self.game, self.lx, self.rng, self.B, self.B_total,
                             value, ms_step, clock_mhz, totals)
        if self.B_total == self.B and not self.args.no_per_config:
            out["per_config"] = measure_per_config(self, value, ms_step, totals, out)
        return out

    def close(self):
        if self.world_size > 1:
            self.dist.destroy_process_group()


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.stub:                                      # CPU test arm (gloo)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from bench_stub import StubArm
        run_distributed(args, StubArm(args))
        return
    run_distributed(args, GpuArm(args))


def native_rollout(game, state, B, max_turns, seed, first, stats, work):
    import ctypes

    from paper_2506_22609_b200 import native
    stuck = ctypes.c_int64(-1)
    native.check(native.lib().lx_rollout(
        game.handle, state.words.data_ptr(), B, int(max_turns), 1 | 2, int(seed), None,
        int(first), stats.data_ptr(), work.data_ptr(), None, None, 0, ctypes.byref(stuck),
        game._stream()))


def measure_e2e(args, game, rng, B, B_total, first, ws, steps=None):
    """e2e through the public API on every rank (each on its own env shard,
    global indices [first, first + B)): Σ env steps over ranks ÷ max over
    ranks of the host wall time of the timed steps, barrier on both sides."""
    import torch
    import torch.distributed as dist

    from paper_2506_22609_b200 import shard
    # ---- e2e: every step copies its episode's per-env seeds host -> device
    # (pinned), runs the fused rollout through the public API and copies the
    # per-env outcomes + the step's stats device -> host.  Steps are
    # double-buffered over three streams (H2D, compute, D2H), so step i+1's
    # upload and step i's download overlap step i's / i+1's rollout; all the
    # copies stay inside the timed region.
    K = steps if steps is not None else max(3, min(args.steps, 30))
    WU = 2
    n_it = K + WU
    seeds_h = [torch.from_numpy(rng.spawn_seeds(rng.episode_seed(0, B_total, 20000 + e), B, first)
                                .view("int64")).pin_memory() for e in range(n_it)]
    seeds_d = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
    outc_d = [torch.empty(B, dtype=torch.int8, device="cuda") for _ in range(2)]
    stats_d = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(2)]
    work_d = [torch.zeros(16, dtype=torch.int64, device="cuda") for _ in range(2)]
    states = [game.empty_state(B) for _ in range(2)]
    outc_h = [torch.empty(B, dtype=torch.int8).pin_memory() for _ in range(n_it)]
    stats_h = [torch.zeros(8, dtype=torch.int64).pin_memory() for _ in range(n_it)]
    s_h2d, s_run, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()                                    # noqa: E731
    h_done = [ev() for _ in range(2)]
    k_done = [ev() for _ in range(2)]
    d_done = [ev() for _ in range(2)]
    for e in k_done + d_done:
        e.record(torch.cuda.current_stream())
    torch.cuda.synchronize()

    def step(it):
        b = it % 2
        with torch.cuda.stream(s_h2d):
            s_h2d.wait_event(k_done[b])             # the rollout that read seeds_d[b] is done
            seeds_d[b].copy_(seeds_h[it], non_blocking=True)
            h_done[b].record(s_h2d)
        with torch.cuda.stream(s_run):
            s_run.wait_event(h_done[b])
            s_run.wait_event(d_done[b])             # outputs of buffer b were downloaded
            game.rollout(seeds=seeds_d[b], out=states[b], max_turns=args.max_turns, store=True,
                         truncate=True, check=False, stats=stats_d[b], work=work_d[b],
                         outcomes=outc_d[b])
            k_done[b].record(s_run)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(k_done[b])
            outc_h[it].copy_(outc_d[b], non_blocking=True)
            stats_h[it].copy_(stats_d[b], non_blocking=True)
            d_done[b].record(s_d2h)
    for it in range(WU):
        step(it)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for it in range(WU, n_it):
        step(it)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if ws > 1:
        dist.barrier()
    steps_done = sum(int(stats_h[it][0]) for it in range(WU, n_it))
    t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    n = torch.tensor([steps_done], dtype=torch.int64, device="cuda")
    shard.max_over_ranks(t)
    shard.reduce_stats(n)
    return {"value": int(n.item()) / float(t.item()), "unit": UNIT,
            "h2d_bytes_per_step": B * 8 * ws, "d2h_bytes_per_step": (B + 64) * ws,
            "steps_timed": K,
            "path": "B200Game.rollout(seeds=host->device) + outcomes/stats device->host, "
                    "double-buffered over H2D / compute / D2H streams, every rank on its "
                    "own shard, max wall time over ranks"}


_PCIE_GBS = None


def pcie_h2d_gbs():
    """Pinned host -> device copy bandwidth of this GPU's link (64 MiB, 10
    copies, CUDA events), measured once per process: the peak of the e2e
    legs' roofline (their bound is the per-env seed upload)."""
    global _PCIE_GBS
    if _PCIE_GBS is None:
        import torch
        n = 64 << 20
        h = torch.empty(n, dtype=torch.uint8).pin_memory()
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        _PCIE_GBS = 10 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    return _PCIE_GBS


def e2e_roofline(e2e, env_steps_per_step, kernel_value, ws=1):
    """Roofline of an e2e leg: the slower of the device rollout (the
    device-timed value of the same config) and the host->device upload of the
    per-env seeds (8 B per env per episode) at the measured PCIe bandwidth."""
    if not isinstance(e2e, dict) or not env_steps_per_step or not kernel_value:
        return None
    pcie = pcie_h2d_gbs() * ws
    per_step = e2e["h2d_bytes_per_step"] / env_steps_per_step
    pcie_bound = pcie * 1e9 / per_step
    bound = min(kernel_value, pcie_bound)
    return {"bound": "pcie_h2d" if pcie_bound < kernel_value else "device_rollout",
            "achieved": e2e["value"], "peak": bound, "unit": UNIT, "frac": e2e["value"] / bound,
            "device_rollout_env_steps_per_s": kernel_value,
            "pcie_h2d": {"peak_gbs": pcie, "achieved_gbs": e2e["value"] * per_step / 1e9,
                         "h2d_bytes_per_env_step": per_step,
                         "bound_env_steps_per_s": pcie_bound,
                         "peak_source": f"pinned host->device copy of 64 MiB in this run, "
                                        f"x{ws} GPUs"}}


def measure_e2e_host(args, game, rng, B, B_total, first, ws, steps=None):
    """e2e through the C-ABI host-buffer calls lx_playout_host_async / _wait
    (what a numpy / ctypes binding of the reference's benchmark loop calls,
    evaluation.py:197-233): every step passes its episode's per-env seeds in
    pinned host memory and gets the per-env outcomes and the stats back in
    host memory; two episodes in flight, so step i+1's seed upload and step
    i-1's download overlap step i's rollout (the native runtime's own three
    streams).  Σ env steps over ranks ÷ max over ranks of the host wall time."""
    import torch
    import torch.distributed as dist

    from paper_2506_22609_b200 import shard
    K = steps if steps is not None else max(3, min(args.steps, 30))
    WU = 2
    n_it = K + WU
    seeds_h = [torch.from_numpy(rng.spawn_seeds(rng.episode_seed(0, B_total, 30000 + e), B, first)
                                .view("int64")).pin_memory() for e in range(n_it)]
    outc_h = [torch.empty(B, dtype=torch.int8).pin_memory() for _ in range(n_it)]
    stats_h = [torch.zeros(8, dtype=torch.int64).pin_memory() for _ in range(n_it)]

    def run(lo, hi):
        # the host stays two episodes ahead: episode i is issued once i-2's
        # outputs are home, so i's upload can start as soon as i-2's rollout
        # (same device slot) has read its seeds
        pending = []
        for it in range(lo, hi):
            pending.append(game.playout_host_async(seeds=seeds_h[it], outcomes=outc_h[it],
                                                   stats=stats_h[it], max_turns=args.max_turns,
                                                   truncate=True))
            if len(pending) > 2:
                game.playout_host_wait(pending.pop(0))
        for t in pending:
            game.playout_host_wait(t)
    run(0, WU)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    run(WU, n_it)
    e2e_s = time.perf_counter() - t0
    if ws > 1:
        dist.barrier()
    steps_done = sum(int(stats_h[it][0]) for it in range(WU, n_it))
    t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    n = torch.tensor([steps_done], dtype=torch.int64, device="cuda")
    shard.max_over_ranks(t)
    shard.reduce_stats(n)
    return {"value": int(n.item()) / float(t.item()), "unit": UNIT,
            "h2d_bytes_per_step": B * 8 * ws, "d2h_bytes_per_step": (B + 64) * ws,
            "steps_timed": K,
            "path": "lx_playout_host_async / _wait (C-ABI, host buffers): pinned host seeds "
                    "in, host outcomes + stats out, the host two episodes ahead (upload, "
                    "rollout and download on the runtime's three streams, two device slots)"}


def rollout_roofline(game, value, totals, clock_mhz):
    """Roofline of the fused rollout kernel: integer ALU pipe bound.
    Per-env-step instruction counts come from the ncu capture of this exact
    cubin (profiles/rollout_<Game>.json, keyed by the NVRTC cache key);
    achieved = count x live env steps/s; peak = pipe rate x SMs x clock."""
    prof = load_profile(game)
    clk_mhz = float(clock_mhz or 1965.0)
    sms = int((prof or {}).get("sms") or 148)
    # ALU pipe peak per SM per cycle from ncu (sm__inst_executed_pipe_alu
    # .avg.peak_sustained: 4 SMSP x 0.5 warp-inst/clk) when the capture has it
    per_sm = float((prof or {}).get("alu_peak_per_sm_cycle") or 2.0)
    src = ("ncu sm__inst_executed_pipe_alu.avg.peak_sustained"
           if (prof or {}).get("alu_peak_per_sm_cycle") else "4 SMSP x 0.5/clk pipe rate")
    peak_alu = sms * per_sm * clk_mhz * 1e6
    peak_issue = sms * 4 * 1.0 * clk_mhz * 1e6        # issue: 1 warp-inst/clk/SMSP
    mean_plies = totals[0] / max(totals[5], 1)
    rl = {"bound": "int_alu", "unit": "Gwarp-inst/s", "kernel": "lx_rollout",
          "peak": peak_alu / 1e9,
          "peak_source": f"{sms} SMs x {per_sm:g} ALU warp-inst/clk/SM ({src}) x "
                         f"{clk_mhz:.0f} MHz SM clock sampled in the run",
          "achieved": None, "frac": None, "traffic": None,
          "algorithmic_bytes_per_env_step": game.info["nq"] * 16 / mean_plies}
    if prof:
        ach = prof["alu_warp_inst_per_env_step"] * value
        iss = prof["warp_inst_per_env_step"] * value
        rl.update({"achieved": ach / 1e9, "frac": ach / peak_alu,
                   "traffic": prof["dram_bytes_per_launch"] / prof["env_steps_in_launch"],
                   "traffic_unit": "DRAM bytes per env step (ncu)",
                   "traffic_bytes_per_launch": prof["dram_bytes_per_launch"],
                   "traffic_profile_batch": prof.get("batch"),
                   "alu_warp_inst_per_env_step": prof["alu_warp_inst_per_env_step"],
                   "issue": {"achieved": iss / 1e9, "peak": peak_issue / 1e9,
                             "frac": iss / peak_issue},
                   "ncu_alu_pipe_pct": prof.get("alu_pipe_elapsed_pct"),
                   "inst_source": prof.get("source"), "cubin_key": prof.get("cubin_key"),
                   "profile_stale": prof.get("stale", False)})
    return rl


def measure_extras(args, game, lx, rng, B, B_total, value, ms_step, clock_mhz, totals):
    """The HBM-bound step kernel, roofline data, the PGX env path and the CPU
    baseline (rank 0, N=1 sizes)."""
    import torch
    out = {"roofline": rollout_roofline(game, value, totals, clock_mhz)}

    # ---- HBM-bound per-ply step kernel (CompiledGame.random_actions + step_into)
    st = game.init(B, seed=1)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    plies = 8
    ev0.record()
    for _ in range(plies):
        game.random_step(st, max_turns=args.max_turns)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / plies
    nbytes = 2 * game.info["nq"] * 16 * B            # read + write the state words
    gbs = nbytes / (ms / 1e3) / 1e9
    peak_hbm = measured_hbm()
    out["step_kernel"] = {"kernel": "lx_random_step", "plies_timed": plies,
                          "ms_per_ply": ms, "env_steps_per_s_upper": B / (ms / 1e3),
                          "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak_hbm,
                                       "unit": "GB/s", "frac": gbs / peak_hbm,
                                       "traffic": step_traffic(game, "lx_random_step", B),
                                       "traffic_unit": "DRAM bytes per launch (ncu, scaled "
                                                       "to this batch)",
                                       "bytes_per_env_ply": 2 * game.info["nq"] * 16}}
    out["env_step_api"] = measure_env_api(args, game, lx, B)
    out["e2e_reference_layout"] = measure_e2e_reference_layout(args, game, lx, rng, B, B_total)

    # ---- CPU baseline (oracle port, all host threads, bounded sample): N=1 only
    if B_total != B:
        return out
    threads = os.cpu_count() or 1
    r, steps, dt, n = cpu_rate(args.game, B_total, args.cpu_seconds, threads, args.max_turns)
    out["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": threads, "kind": "port",
                           "cpu_model": cpu_model(),
                           "sample": f"{steps} env steps, first {n} envs of episode 10000, "
                                     f"{dt:.1f}s on {threads} threads"}
    return out


def measure_e2e_reference_layout(args, game, lx, rng, B, B_total, steps=5):
    """The drop-in call end to end: engine.playout_random(game, seed, B)
    (engine.py:123-163) with the final states exported to host numpy arrays
    in the reference GameState layout (state.py:78-130) every step -- one
    fused rollout, one lx_export, one device-to-host copy of every reference
    field.  Host wall time, synchronised."""
    import torch
    lx.engine.playout_random(game, seed=1, batch_size=B).final.host()     # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    steps_done, d2h = 0, 0
    po = host = None
    for e in range(steps):
        po = host = None                    # the caller is done with the previous result
        po = lx.engine.playout_random(game, seed=rng.episode_seed(0, B_total, 30_000 + e),
                                      batch_size=B, max_turns=args.max_turns)
        host = po.final.host()
        steps_done += int(po.stats[0])
        d2h = sum(v.nbytes for v in host.values())
    dt = time.perf_counter() - t0
    return {"value": steps_done / dt, "unit": UNIT, "h2d_bytes_per_step": 8,
            "d2h_bytes_per_step": d2h, "steps_timed": steps,
            "path": "engine.playout_random(game, seed, B).final.host(): fused rollout + "
                    "lx_export + device->host copy of every reference GameState field "
                    f"({d2h // B} B/env), host wall time"}


def measure_env_api(args, game, lx, B):
    """PGX-style API path (LudaxEnvironment): one fused launch per ply
    (uniform-random action sampled in the step kernel, auto-reset), device
    tensors, output buffers reused; bool mask and bit-packed mask variants."""
    import torch
    peak_hbm = measured_hbm()
    res = {}
    for fmt in ("bool", "bits"):
        env = lx.LudaxEnvironment(game, auto_reset=True, mask_format=fmt)
        est = env.init(seed=2, batch_size=B)
        for _ in range(16):
            est = env.step_(est, env.RANDOM)
        torch.cuda.synchronize()
        plies = 64
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(plies):
            est = env.step_(est, env.RANDOM)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / plies
        b_env = env.bytes_per_env_step()
        gbs = b_env * B / (ms / 1e3) / 1e9
        res[fmt] = {"env_steps_per_s": B / (ms / 1e3), "ms_per_ply": ms,
                    "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak_hbm,
                                 "unit": "GB/s", "frac": gbs / peak_hbm,
                                 "traffic": step_traffic(game, "lx_env_step", B, fmt),
                                 "traffic_unit": "DRAM bytes per launch (ncu, scaled to "
                                                 "this batch)",
                                 "bytes_per_env_step": b_env}}
    return {"path": "LudaxEnvironment.step_(state, RANDOM) (auto_reset): action sampled, "
                    "applied, rewards / flags / next legal mask written in one lx_env_step "
                    "launch per ply; device tensors, output buffers reused",
            "kernel": "lx_env_step", "plies_timed": 64,
            "env_steps_per_s": res["bool"]["env_steps_per_s"],
            "roofline": res["bool"]["roofline"], "bits_mask": res["bits"]}


# ------------------------------------------------------------------ per-config block
def time_config(arm, game, B, steps, warmup, max_turns):
    """Timed episodes of one config on this GPU (N=1): returns (ms, totals,
    final-state buffer of the last timed episode, its episode id)."""
    torch, rng = arm.torch, arm.rng
    state = game.empty_state(B)
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    work = torch.zeros(16, dtype=torch.int64, device="cuda")
    acc = torch.zeros(8, dtype=torch.int64, device="cuda")

    def ep(e):
        native_rollout(game, state, B, max_turns, rng.episode_seed(0, B, e), 0, stats, work)
        acc.add_(stats)
    for w in range(warmup):
        ep(w)
    torch.cuda.synchronize()
    acc.zero_()
    graph = None
    if B <= GRAPH_MAX_BATCH:
        # launch-bound sizes: the K timed episodes (each its own seed) are
        # captured once into a CUDA graph and replayed as one launch; each
        # episode publishes its stats into its own row (summed after the
        # timed region), so the graph holds only lx_rollout nodes
        per_ep = torch.zeros(steps, 8, dtype=torch.int64, device="cuda")
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for e in range(steps):
                native_rollout(game, state, B, max_turns, rng.episode_seed(0, B, 10_000 + e), 0,
                               per_ep[e], work)
        # warm replays for >= 50 ms: the timed replay is a few ms, so the SM
        # clock must already be up when it starts
        t_warm, n_warm = time.perf_counter(), 0
        while time.perf_counter() - t_warm < 0.05:
            graph.replay()
            torch.cuda.synchronize()
            n_warm += 1
        # the timed region repeats the replay for >= 0.25 s so the clock
        # sampler sees it (the episodes read no input but their seeds)
        reps = max(1, int(0.25 / ((time.perf_counter() - t_warm) / n_warm)) + 1)
    else:
        reps = 1
    run = ((lambda: [graph.replay() for _ in range(reps)]) if graph is not None
           else (lambda: [ep(10_000 + e) for e in range(steps)]))
    with ClockSampler(arm.local) as clk:
        ms = arm.timed(run) / reps
    if graph is not None:
        acc.copy_(per_ep.sum(0))
    return ms, acc.cpu().tolist(), state, 10_000 + steps - 1, clk.summary(), graph is not None


def parity_check(name, game, state, B, episode, n, max_turns):
    """Every field of the first n final states of the benchmarked episode
    (exported to the reference GameState layout by lx_export) against the
    CPU oracle replaying the same env seeds; also the oracle's rate on that
    sample (the config's cpu_baseline).  The bench episodes do not truncate
    (reference _run_episode); the cap's truncation is applied to both sides
    the way engine.playout_random does (engine.py:156-160)."""
    import numpy as np

    from oracle import oracle as O
    from paper_2506_22609_b200.game import DeviceState
    n = min(n, B)
    sub = DeviceState(game, state.words[:, :n].contiguous(), n) if n < B else state
    got = game._export(sub)
    cap = ~got["terminated"]
    got["terminated"] = got["terminated"] | cap
    got["truncated"] = got["truncated"] | cap
    got["outcome"] = np.where(cap, 0, got["outcome"]).astype(np.int8)
    og = O.OracleGame(name)
    threads = os.cpu_count() or 1
    seeds = O.spawn_seeds(O.hash_key3(0, B, episode), n)
    st = og.init(n, seeds=seeds)
    t0 = time.perf_counter()
    want, steps = og.playout(state=st, max_turns=max_turns, threads=threads)
    dt = time.perf_counter() - t0
    bad = np.zeros(n, bool)
    fields = []
    for k, v in want.items():
        if k not in got:
            continue
        fields.append(k)
        a, b = np.asarray(got[k]).reshape(n, -1), np.asarray(v).reshape(n, -1)
        bad |= (a != b).any(axis=1)
    first_bad = int(np.argmax(bad)) if bad.any() else None
    return ({"envs_checked": n, "of_batch": B, "episode": episode, "mismatches": int(bad.sum()),
             "first_mismatch_row": first_bad, "fields": fields,
             "checker": "oracle/ludax_oracle.c (C restatement pinned to reference fixtures)"},
            {"value": steps / dt, "unit": UNIT, "cores": threads, "kind": "port",
             "cpu_model": cpu_model(),
             "sample": f"the first {n} envs of benchmarked episode {episode} replayed by the "
                       f"oracle port for the parity check: {steps} env steps, {dt:.1f}s on "
                       f"{threads} threads"})


def measure_per_config(arm, value, ms_step, totals, head_extras):
    """Every BASELINE.json config at N=1 (see PER_CONFIG)."""
    args = arm.args
    out = []
    for label, name, B, steps, n_par in PER_CONFIG:
        n_par = max(1, int(n_par * args.parity_scale))
        entry = {"config": label, "game": name, "batch": B}
        if name == args.game and B == args.batch:
            # the headline: its timed episodes, e2e and roofline are the line's own
            game, state, episode = arm.game, arm.state, arm.last_episode
            entry.update({"steps": args.steps, "ms_per_step": ms_step, "value": value,
                          "mean_plies": totals[0] / max(totals[5], 1),
                          "roofline": head_extras.get("roofline"), "e2e": "headline e2e",
                          "clocks": "headline clocks"})
        else:
            game = arm.lx.load_config_game(name)
            ms, tot, state, episode, clk, graphed = time_config(arm, game, B, steps, 3,
                                                                args.max_turns)
            val = tot[0] / (ms / 1000.0)
            entry.update({"steps": steps, "warmup": 3, "ms_per_step": ms / steps, "value": val,
                          "cuda_graph": graphed,
                          "mean_plies": tot[0] / max(tot[5], 1),
                          "totals": {"env_steps": tot[0], "p1_wins": tot[1], "p2_wins": tot[2],
                                     "draws": tot[3], "envs": tot[5]},
                          "clocks": clk,
                          "roofline": rollout_roofline(game, val, tot, clk.get("sm_mhz")),
                          "e2e": measure_e2e_host(args, game, arm.rng, B, B, 0, 1,
                                                  steps=min(steps, 20)),
                          "e2e_python": measure_e2e(args, game, arm.rng, B, B, 0, 1,
                                             steps=min(steps, 20))})
        if isinstance(entry.get("e2e"), dict):
            per_step = entry["totals"]["env_steps"] / steps
            for k in ("e2e", "e2e_python"):
                rl = e2e_roofline(entry.get(k), per_step, entry.get("value"))
                if rl:
                    entry[k]["roofline"] = rl
        entry["unit"] = UNIT
        entry["workload"] = (f"{GAME_FILES[name]} uniform-random rollouts, {B} envs, "
                             f"full episodes (cap {args.max_turns} plies)")
        par, cpu = parity_check(name, game, state, B, episode, n_par, args.max_turns)
        entry["parity"] = par
        entry["cpu_baseline"] = cpu
        out.append(entry)
    return out


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6553.3


def load_profile(game):
    """Per-env-step instruction count of this exact kernel build, from the
    committed ncu capture (profiles/rollout_<game>.json)."""
    path = os.path.join(ROOT, "profiles", f"rollout_{game.info['name'].replace(' ', '_')}.json")
    try:
        with open(path) as f:
            prof = json.load(f)
    except Exception:
        return None
    # a capture of an older build of this game is still the best available
    # count; say so instead of dropping the roofline
    prof["stale"] = bool(prof.get("cubin_key")) and prof["cubin_key"] != game.lowered_key()
    return prof


def step_traffic(game, kernel, B, variant=None):
    """DRAM bytes of one launch of a per-ply kernel at batch B, from the
    committed ncu --set full capture (profiles/step_<game>.json, written by
    tools/ncu_summary.py from tools/ncu_step.py); None when absent or when it
    was taken on another build of this game."""
    path = os.path.join(ROOT, "profiles", f"step_{game.info['name'].replace(' ', '_')}.json")
    try:
        with open(path) as f:
            prof = json.load(f)
        if prof.get("cubin_key") != game.lowered_key():
            return None
        key = kernel if variant in (None, "bool") else f"{kernel}:{variant}"
        return prof["kernels"][key]["dram_bytes_per_env"] * B
    except Exception:
        return None


if __name__ == "__main__":
    main()
