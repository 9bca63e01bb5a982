"""MCTS match throughput: agents.play_match on the device
path vs the unmodified reference (baseline/_ref) on the same seeds, plus a
check that both produce identical MatchStats.

    python tools/mcts_bench.py [--game connect_four] [--games 16] [--strong 100]
                               [--weak 50] [--no-reference] [--gavel --matches 100]

Prints one JSON line: wall seconds and MCTS iterations/s of each side.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

p = argparse.ArgumentParser()
p.add_argument("--game", default="connect_four")
p.add_argument("--games", type=int, default=16)
p.add_argument("--strong", type=int, default=100)
p.add_argument("--weak", type=int, default=50)
p.add_argument("--seed", type=int, default=0)
p.add_argument("--no-reference", action="store_true")
p.add_argument("--gavel", action="store_true",
               help="time evaluation.evaluate_game (GAVEL report) instead of one match")
p.add_argument("--matches", type=int, default=100)
a = p.parse_args()

text = open(os.path.join(ROOT, "paper_2506_22609_b200", "games", f"{a.game}.ldx")).read()


def stats_key(st):
    return (st.wins_p1, st.wins_p2, st.draws, st.truncations, st.turns.tolist(),
            st.legal_counts.tolist(), st.winner_agent.tolist())


def iterations(st):
    # every decision of seat A costs `strong` iterations, of seat B `weak`
    return int(st.total_turns) * (a.strong + a.weak) / 2


import torch  # noqa: E402
import paper_2506_22609_b200 as lx  # noqa: E402
from paper_2506_22609_b200 import agents  # noqa: E402

if a.gavel:
    from paper_2506_22609_b200 import evaluation  # noqa: E402
    cfg = dict(matches=a.matches, strong_iterations=a.strong, weak_iterations=a.weak, seed=a.seed)
    lx.load_game(text).native                          # CUDA context + NVRTC cache warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = evaluation.evaluate_game(text, evaluation.EvalConfig(**cfg)).as_dict()
    t_mine = time.perf_counter() - t0
    out = {"game": a.game, "gavel": cfg, "b200": {"seconds": t_mine}, "report": rep}
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not a.no_reference and os.path.isdir(os.path.join(ref_dir, "boardlang")):
        sys.path.insert(0, ref_dir)
        from boardlang import evaluation as revaluation  # noqa: E402
        t0 = time.perf_counter()
        rrep = revaluation.evaluate_game(text, revaluation.EvalConfig(**cfg)).as_dict()
        t_ref = time.perf_counter() - t0
        out["reference"] = {"seconds": t_ref, "cores": 1}
        out["identical_report"] = rrep == rep
        out["speedup"] = t_ref / t_mine
    print(json.dumps(out))
    sys.exit(0)

g = lx.load_game(text)
strong = agents.MctsPolicy(agents.MctsConfig(iterations=a.strong, seed=a.seed * 2 + 1))
weak = agents.MctsPolicy(agents.MctsConfig(iterations=a.weak, seed=a.seed * 2 + 2))
agents.play_match(g, agents.MctsPolicy(iterations=4), agents.MctsPolicy(iterations=2), 2)  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
mine = agents.play_match(g, strong, weak, a.games, seed=a.seed)
torch.cuda.synchronize()
t_mine = time.perf_counter() - t0
out = {"game": a.game, "games": a.games, "strong": a.strong, "weak": a.weak,
       "plies": int(mine.total_turns),
       "b200": {"seconds": t_mine, "iterations_per_s": iterations(mine) / t_mine}}
ref_dir = os.path.join(ROOT, "baseline", "_ref")
if not a.no_reference and os.path.isdir(os.path.join(ref_dir, "boardlang")):
    sys.path.insert(0, ref_dir)
    import boardlang  # noqa: E402
    from boardlang import agents as ragents  # noqa: E402
    rg = boardlang.load_game(text)
    rs = ragents.MctsPolicy(ragents.MctsConfig(iterations=a.strong, seed=a.seed * 2 + 1))
    rw = ragents.MctsPolicy(ragents.MctsConfig(iterations=a.weak, seed=a.seed * 2 + 2))
    t0 = time.perf_counter()
    ref = ragents.play_match(rg, rs, rw, a.games, seed=a.seed)
    t_ref = time.perf_counter() - t0
    out["reference"] = {"seconds": t_ref, "iterations_per_s": iterations(ref) / t_ref,
                        "cores": 1}
    out["identical_stats"] = stats_key(ref) == stats_key(mine)
    out["speedup"] = t_ref / t_mine
print(json.dumps(out))
