"""Summarise ncu reports of lx_rollout into profiles/ (run locally, no GPU).

    python tools/ncu_summary.py gpurun_out --tag r1 [--out profiles]

Reads gpurun_out/prof_<game>.ncu-rep (+ plain_<game>.json written by
tools/ncu_rollout.py for the env-step count of the profiled launch) and
writes profiles/<tag>_rollout_<game>.json plus profiles/rollout_<Game>.json
(the file bench.py reads for the per-env-step instruction count).
"""
import argparse
import csv
import io
import json
import os
import subprocess

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "smsp__inst_executed.sum": "warp_inst",
    "thread_inst_executed": "thread_inst",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed": "alu_pipe_elapsed_pct",
    "device__attribute_multiprocessor_count": "sms",
    "sm__inst_executed_pipe_fma.sum": "fma_warp_inst",
    "sm__inst_executed_pipe_alu.sum": "alu_warp_inst_counted",
    "sm__inst_executed_pipe_alu.avg.peak_sustained": "alu_peak_per_sm_cycle",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_lanes_per_inst",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio": "stall_branch",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
}
UNITS = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1e3, "ms": 1e6,
         "ns": 1.0, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for k, name in METRICS.items():
        if k in head:
            i = head.index(k)
            v = float(vals[i].replace(",", ""))
            res[name] = v * UNITS.get(units[i], 1.0)
    return res


def step_summaries(a):
    """gpurun_out/step_<game>.json (tools/ncu_step.py) + stepprof_<game>_<kernel>.ncu-rep
    -> profiles/<tag>_step_<game>.json and profiles/step_<Game>.json (read by bench.py
    for the `traffic` of the HBM-bound per-ply kernels)."""
    for fn in sorted(os.listdir(a.src)):
        if not (fn.startswith("step_") and fn.endswith(".json")):
            continue
        with open(os.path.join(a.src, fn)) as f:
            info = json.loads(f.read().strip().splitlines()[-1])
        game, B = info["game"], info["batch"]
        out = {"game": game, "batch": B, "cubin_key": info["cubin_key"], "kernels": {}}
        for k in ("lx_random_step", "lx_env_step", "lx_env_step_bits"):
            rep = os.path.join(a.src, f"stepprof_{game}_{k}.ncu-rep")
            if not os.path.exists(rep):
                continue
            m = raw(rep)
            dram = m.get("dram_read", 0) + m.get("dram_write", 0)
            out["kernels"][k.replace("_bits", ":bits")] = {
                "duration_ns": m["duration_ns"], "dram_read": m.get("dram_read", 0),
                "dram_write": m.get("dram_write", 0), "dram_bytes_per_env": dram / B,
                "dram_gbs_under_ncu": dram / m["duration_ns"],
                "registers": m.get("registers"), "grid": m.get("grid"),
                "source": f"ncu --set full, {os.path.basename(rep)} (serialised, cold cache)"}
            print(game, k, f"{dram / B:.1f} DRAM B/env", f"{dram / m['duration_ns']:.0f} GB/s")
        from paper_2506_22609_b200.game import GAMES_DIR
        from paper_2506_22609_b200.syntax import parse_game
        with open(os.path.join(GAMES_DIR, f"{game}.ldx")) as f:
            gname = parse_game(f.read()).name.replace(" ", "_")
        for path in (os.path.join(a.out, f"{a.tag}_step_{game}.json"),
                     os.path.join(a.out, f"step_{gname}.json")):
            with open(path, "w") as f:
                json.dump(out, f, indent=1, sort_keys=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("src")
    p.add_argument("--tag", default="r1")
    p.add_argument("--out", default="profiles")
    a = p.parse_args()
    os.makedirs(a.out, exist_ok=True)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    step_summaries(a)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2506_22609_b200.game import GAMES_DIR
    from paper_2506_22609_b200.syntax import parse_game
    names = {}
    for fn in sorted(os.listdir(GAMES_DIR)):
        if fn.endswith(".ldx"):
            with open(os.path.join(GAMES_DIR, fn)) as f:
                names[fn[:-4]] = parse_game(f.read()).name.replace(" ", "_")
    for game, gname in names.items():
        rep = os.path.join(a.src, f"prof_{game}.ncu-rep")
        plain = os.path.join(a.src, f"plain_{game}.json")
        if not (os.path.exists(rep) and os.path.exists(plain)):
            continue
        with open(plain) as f:
            info = json.loads(f.read().strip().splitlines()[-1])
        m = raw(rep)
        steps = info["env_steps"]
        # ALU pipe: 0.5 warp-inst/clk per SMSP, 4 SMSPs per SM (B300_MICROARCH.md)
        sms = m.get("sms", 148)
        if "alu_warp_inst_counted" in m:       # direct count (ncu sm__inst_executed_pipe_alu)
            m["alu_warp_inst"] = m["alu_warp_inst_counted"]
        else:                                  # pipe utilisation x ncu's 0.5/clk/SMSP rate
            m["alu_warp_inst"] = (m.get("alu_pipe_elapsed_pct", 0) / 100.0 * 0.5 * 4 * sms
                                  * m["sm_clock_hz"] * m["duration_ns"] / 1e9)
        s = {"game": game, "batch": info["batch"], "cubin_key": info["cubin_key"],
             "env_steps_in_launch": steps, **m,
             "warp_inst_per_env_step": m["warp_inst"] / steps,
             "thread_inst_per_env_step": m.get("thread_inst", 0) / steps,
             "alu_warp_inst_per_env_step": m.get("alu_warp_inst", 0) / steps,
             "dram_bytes_per_launch": m.get("dram_read", 0) + m.get("dram_write", 0),
             "env_steps_per_s_under_ncu": steps / (m["duration_ns"] / 1e9),
             "source": f"ncu --set full, {os.path.basename(rep)} (serialised, cold cache)"}
        with open(os.path.join(a.out, f"{a.tag}_rollout_{game}.json"), "w") as f:
            json.dump(s, f, indent=1, sort_keys=True)
        with open(os.path.join(a.out, f"rollout_{gname}.json"), "w") as f:
            json.dump(s, f, indent=1, sort_keys=True)
        print(game, f"{s['warp_inst_per_env_step']:.2f} warp-inst/step",
              f"lanes {m.get('active_lanes_per_inst', 0):.1f}",
              f"alu {m.get('alu_pipe_pct', 0):.1f}%", f"issue {m.get('issue_active_pct', 0):.1f}%",
              f"{s['env_steps_per_s_under_ncu'] / 1e9:.1f} G/s")


if __name__ == "__main__":
    main()
