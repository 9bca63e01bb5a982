"""Generate tests/golden/ fixtures FROM THE REFERENCE ITSELF (test infra only).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

The fixtures pin the oracle (oracle/ludax_oracle.c) and the device path to
the reference's exact behaviour; the GPU box never needs /root/reference.
Every fixture below is produced by the reference's public API:
``engine.playout_random`` (engine.py:123-163), ``CompiledGame.legal_mask`` /
``step`` (compiler.py:411-454), ``rng.hash_key`` / ``uniform`` (rng.py:26-42),
``GameState.digest`` (state.py:180-188), and ``parser.parse_game``.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

REF = os.environ.get("LUDAX_REFERENCE", "/root/reference/pkg")
sys.path.insert(0, os.path.join(REF, "src"))

import boardlang  # noqa: E402
from boardlang import engine, rng  # noqa: E402
from boardlang.parser import parse_game  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
GAMES_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "paper_2506_22609_b200", "games")
GAMES = ("tic_tac_toe", "connect_four", "hex", "reversi", "pente", "gomoku", "yavalath",
         "english_draughts", "dai_hasami_shogi", "wolf_and_sheep", "gridworld")
PLAYOUT = {"tic_tac_toe": [(1024, 0), (512, 99)], "connect_four": [(256, 0), (256, 5)],
           "hex": [(64, 0), (48, 21)], "reversi": [(64, 0), (64, 12)],
           "pente": [(32, 0), (24, 3)], "gomoku": [(32, 0), (24, 5)],
           "yavalath": [(128, 0), (96, 9)],
           "english_draughts": [(64, 0), (48, 7)], "dai_hasami_shogi": [(32, 0), (24, 4)],
           "wolf_and_sheep": [(128, 0), (64, 8)], "gridworld": [(256, 0), (128, 3)]}


def state_arrays(st, prefix):
    out = {}
    for name in ("board_piece", "board_owner", "current_player", "move_count", "terminated",
                 "truncated", "outcome", "seeds", "scores", "pass_streak", "pass_flags",
                 "must_move", "last_mover", "last_kind", "last_source", "last_dest",
                 "last_dest_by_player", "hopped_mask", "captured_mask", "promoted_mask",
                 "comp_labels", "phase", "turn_pos"):
        v = getattr(st, name)
        if v is not None:
            out[f"{prefix}{name}"] = v
    return out


def norm(x):
    if dataclasses.is_dataclass(x):
        return [type(x).__name__] + [[f.name, norm(getattr(x, f.name))]
                                     for f in dataclasses.fields(x)]
    if isinstance(x, tuple):
        return [norm(i) for i in x]
    return x


def main():
    os.makedirs(OUT, exist_ok=True)
    meta = {"reference": REF, "games": {}}
    for name in GAMES:
        text = open(os.path.join(GAMES_DIR, f"{name}.ldx")).read()
        ref_text = open(os.path.join(REF, "games", f"{name}.ldx")).read()
        g = boardlang.load_game(text)
        assert norm(parse_game(text)) == norm(parse_game(ref_text)), name
        arrays = {}
        info = {"ast": norm(parse_game(text)), "describe": g.describe(), "playouts": []}
        # (1) final states of seeded random playouts
        for k, (B, seed) in enumerate(PLAYOUT[name]):
            po = engine.playout_random(g, seed=seed, batch_size=B, max_turns=200)
            arrays.update(state_arrays(po.final, f"p{k}_"))
            info["playouts"].append({"batch": B, "seed": seed, "digest": po.final.digest(),
                                     "turns": int(po.turns_taken.sum())})
        # (2) a recorded trajectory: legal mask + sampled action per step
        st = g.init(batch_size=4, seed=3)
        masks, actions, digests = [], [], []
        while not st.terminated.all() and len(actions) < 200:
            masks.append(g.legal_mask(st))
            u = rng.uniform(st.seeds, st.move_count.astype(np.uint64))
            a = g.sample_actions(st, u)
            actions.append(a)
            live = ~st.terminated
            g.step_into(st, a, rows=live, verify=False)
            digests.append(st.digest())
        arrays["traj_masks"] = np.packbits(np.stack(masks), axis=-1)
        arrays["traj_actions"] = np.stack(actions)
        info["traj_digests"] = digests
        info["traj_mask_width"] = int(g.codec.size)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
        meta["games"][name] = info
        print(name, "ok", [p["digest"] for p in info["playouts"]])

    # (3) known-answer transcripts from the reference's own tests
    kat = {}
    ttt = boardlang.load_game(open(os.path.join(GAMES_DIR, "tic_tac_toe.ldx")).read())
    s = engine.init(ttt, 1)
    for a in [0, 1, 4, 2, 8]:                       # tests/test_engine.py:46-51
        s = engine.step(ttt, s, a)
    kat["ttt_diag"] = {"actions": [0, 1, 4, 2, 8], "digest": s.digest(),
                       "outcome": int(s.outcome[0])}
    c4 = boardlang.load_game(open(os.path.join(GAMES_DIR, "connect_four.ldx")).read())
    kat["c4_initial_legal"] = np.nonzero(c4.legal_mask(c4.init(1))[0])[0].tolist()
    rv = boardlang.load_game(open(os.path.join(GAMES_DIR, "reversi.ldx")).read())
    kat["reversi_initial_legal"] = np.nonzero(rv.legal_mask(rv.init(1))[0])[0].tolist()
    pe = boardlang.load_game(open(os.path.join(GAMES_DIR, "pente.ldx")).read())
    for key, seq in (("pente_capture", [180, 181, 200, 182, 183]),      # test_compiler.py:182-195
                     ("pente_no_capture3", [180, 181, 220, 182, 221, 183, 184])):
        s = pe.init(1)
        for a in seq:
            s = pe.step(s, np.array([a]))
        kat[key] = {"actions": seq, "digest": s.digest(),
                    "owner": s.board_owner[0].tolist(), "scores": s.scores[0].tolist()}
    # (4) RNG vectors (rng.py) incl. the benchmark's episode keys (evaluation.py:222-229)
    seeds = rng.spawn_seeds(12345, 16)
    mcs = np.arange(16, dtype=np.uint64) * 7
    kat["rng"] = {"spawn_12345_16": [str(int(x)) for x in seeds],
                  "uniform_hex": [float.hex(float(x)) for x in rng.uniform(seeds, mcs)],
                  "episode_keys": {f"{b}_{e}": str(int(rng.hash_key(np.uint64(0), np.uint64(b),
                                                                    np.uint64(e))))
                                   for b in (1024, 1 << 20) for e in (0, 1, 10000, 10001)}}
    # (5) C4 opening distribution (tests/test_agents.py:28-41) and TTT outcome counts
    st = c4.init(batch_size=100_000, seed=77)
    a = c4.sample_actions(st, rng.uniform(st.seeds, st.move_count.astype(np.uint64)))
    vals, cnt = np.unique(a, return_counts=True)
    kat["c4_opening_counts"] = dict(zip(map(str, vals.tolist()), cnt.tolist()))
    f = engine.playout_random(ttt, seed=11, batch_size=10_000).final
    kat["ttt_10000_seed11"] = {"p1": int((f.outcome == 1).sum()),
                               "p2": int((f.outcome == 2).sum()),
                               "draw": int((f.outcome == 0).sum()),
                               "digest": f.digest()}
    # (6) movement transcripts (tests/test_acceptance.py:148-178,
    #     test_engine.py:159-196, test_compiler.py:198-204)
    dr_text = open(os.path.join(GAMES_DIR, "english_draughts.ldx")).read()
    dr = boardlang.load_game(dr_text)
    C = 64
    s = dr.init(1)
    for a in (44 * C + 35, 21 * C + 30, 35 * C + 26):
        s = dr.step(s, np.array([a]))
    kat["draughts_forced"] = {"actions": [44 * C + 35, 21 * C + 30, 35 * C + 26],
                              "legal": np.nonzero(dr.legal_mask(s)[0])[0].tolist(),
                              "digest": s.digest()}
    s = dr.step(s, np.array([17 * C + 35]))
    kat["draughts_forced"]["after_capture"] = {"digest": s.digest(),
                                               "current_player": int(s.current_player[0])}
    drill_text = dr_text.replace("(40 42 44 46 49 51 53 55 56 58 60 62)", "(36 58)").replace(
        "(1 3 5 7 8 10 12 14 17 19 21 23)", "(27 9 14)")
    g = boardlang.load_game(drill_text)
    s = g.init(1)
    drill = {"start_legal": np.nonzero(g.legal_mask(s)[0])[0].tolist()}
    s = g.step(s, np.array([36 * C + 18]))
    drill["after1"] = {"current_player": int(s.current_player[0]),
                       "must_move": int(s.must_move[0]),
                       "legal": np.nonzero(g.legal_mask(s)[0])[0].tolist(), "digest": s.digest()}
    s = g.step(s, np.array([18 * C + 0]))
    drill["after2"] = {"current_player": int(s.current_player[0]),
                       "piece0": int(s.board_piece[0, 0]), "digest": s.digest()}
    drill["text_replace"] = [["(40 42 44 46 49 51 53 55 56 58 60 62)", "(36 58)"],
                             ["(1 3 5 7 8 10 12 14 17 19 21 23)", "(27 9 14)"]]
    kat["draughts_drill"] = drill
    gw = boardlang.load_game(open(os.path.join(GAMES_DIR, "gridworld.ldx")).read())
    s = gw.init(1)
    grid = {"directions": list(gw.codec.directions),
            "initial_legal": np.nonzero(gw.legal_mask(s)[0])[0].tolist()}
    right, down = gw.codec.encode_direction("right"), gw.codec.encode_direction("down")
    s = gw.step(s, np.array([right]))
    s = gw.step(s, np.array([down]))
    grid["right_down"] = {"actions": [int(right), int(down)], "digest": s.digest(),
                          "outcome": int(s.outcome[0]), "terminated": bool(s.terminated[0])}
    kat["gridworld"] = grid
    meta["kat"] = kat
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=0, sort_keys=True)
    print("wrote", OUT)


def _stats_dict(st):
    return {"games": st.games, "wins_p1": st.wins_p1, "wins_p2": st.wins_p2, "draws": st.draws,
            "truncations": st.truncations, "turns": st.turns.tolist(),
            "legal_counts": st.legal_counts.tolist(),
            "multi_choice_turns": st.multi_choice_turns, "total_turns": st.total_turns,
            "coverage": [float.hex(float(x)) for x in st.coverage],
            "seat_of_a": st.seat_of_a.tolist(), "winner_agent": st.winner_agent.tolist(),
            "wins_a": st.wins_a, "wins_b": st.wins_b}


MATCHES = [
    # (game, policy a, policy b, games, seed, max_turns); policy = ("mcts", iters, seed) | ("random", seed)
    ("tic_tac_toe", ("mcts", 30, 1), ("random", 2), 8, 3, 200),
    ("connect_four", ("mcts", 40, 5), ("mcts", 15, 6), 6, 7, 200),
    ("reversi", ("mcts", 12, 1), ("random", 3), 4, 2, 200),
    ("hex", ("mcts", 10, 4), ("mcts", 5, 5), 2, 11, 200),
    ("english_draughts", ("mcts", 12, 2), ("mcts", 6, 3), 4, 4, 60),
    ("wolf_and_sheep", ("random", 7), ("mcts", 10, 8), 4, 5, 200),
]


def mcts_fixtures():
    """MCTS decisions, match statistics and a GAVEL report from the
    reference agents (agents.py, evaluation.py:85-143)."""
    from boardlang.agents import MctsConfig, MctsPolicy, RandomPolicy, mcts_search, play_match
    from boardlang.evaluation import EvalConfig, evaluate_game

    def pol(p):
        return MctsPolicy(MctsConfig(iterations=p[1], seed=p[2])) if p[0] == "mcts" \
            else RandomPolicy(seed=p[1])
    out = {"matches": [], "searches": []}
    for name, a, b, n, seed, mt in MATCHES:
        g = boardlang.load_game(open(os.path.join(GAMES_DIR, f"{name}.ldx")).read())
        st = play_match(g, pol(a), pol(b), n, seed=seed, max_turns=mt)
        from boardlang.evaluation import harmonic_mean, score_match
        sc = score_match(st)
        out["matches"].append({"game": name, "a": list(a), "b": list(b), "games": n,
                               "seed": seed, "max_turns": mt, "stats": _stats_dict(st),
                               "scores": {k: float.hex(v) for k, v in sc.as_dict().items()},
                               "gavel": float.hex(harmonic_mean(sc.values()))})
        print("match", name, st.wins_a, st.wins_b)
    for name, seq, iters, seed in (("connect_four", [38, 39, 31], 300, 9),
                                   ("tic_tac_toe", [4], 200, 3),
                                   ("reversi", [19], 80, 5),
                                   ("english_draughts", [44 * 64 + 35, 21 * 64 + 30], 60, 2)):
        g = boardlang.load_game(open(os.path.join(GAMES_DIR, f"{name}.ldx")).read())
        s = g.init(1, seed=13)
        for a in seq:
            s = g.step(s, np.array([a]))
        act = mcts_search(g, s, MctsConfig(iterations=iters, seed=seed))
        out["searches"].append({"game": name, "actions": seq, "iterations": iters,
                                "seed": seed, "init_seed": 13, "best": int(act)})
        print("search", name, act)
    rep = evaluate_game(open(os.path.join(GAMES_DIR, "tic_tac_toe.ldx")).read(),
                        EvalConfig(matches=6, strong_iterations=20, weak_iterations=8, seed=1))
    out["gavel_ttt"] = {"config": {"matches": 6, "strong_iterations": 20, "weak_iterations": 8,
                                   "seed": 1}, "report": rep.as_dict()}
    with open(os.path.join(OUT, "mcts.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print("wrote mcts.json")


def jsonl_fixtures():
    """Recorded trajectories in the reference's JSONL wire format
    (Playouts.to_jsonl, engine.py:90-120) plus the final digests."""
    out = {}
    for name, seed, B in (("tic_tac_toe", 5, 3), ("reversi", 6, 2), ("english_draughts", 7, 2),
                          ("gridworld", 8, 3), ("pente", 9, 1)):
        g = boardlang.load_game(open(os.path.join(GAMES_DIR, f"{name}.ldx")).read())
        po = engine.playout_random(g, seed=seed, batch_size=B, record=True)
        out[name] = {"seed": seed, "batch": B, "jsonl": [po.to_jsonl(i) for i in range(B)],
                     "digest": po.final.digest()}
    with open(os.path.join(OUT, "jsonl.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print("wrote jsonl.json")


def fuzz_fixtures(corpora=((7, 5, 150), (11, 6, 120), (23, 8, 150), (31, 10, 150)), tries=20000):
    """Programs from the reference's own random generator (generator.py,
    sample_game; sampler seeds 7, 11, 23, 31 at depths 5, 6, 8, 10) that the reference compiles and
    plays (playout_random, B=16, 60-ply cap) -- a corpus for checking the
    lowering's generality: every one must either be lowered bit-exactly or
    rejected with CompileError."""
    import signal
    from boardlang.generator import SamplerConfig, sample_game

    class _Timeout(Exception):
        pass

    def _alarm(*_):
        raise _Timeout()
    signal.signal(signal.SIGALRM, _alarm)
    out = []
    for sampler_seed, depth, limit in corpora:
        out += _fuzz_corpus(sampler_seed, depth, limit, tries, _Timeout)
    with open(os.path.join(OUT, "fuzz.json"), "w") as fh:
        json.dump({"batch": 16, "max_turns": 60, "programs": out}, fh, indent=0, sort_keys=True)
    print("wrote fuzz.json", len(out))


def _fuzz_corpus(sampler_seed, depth, limit, tries, timeout_exc):
    from boardlang.generator import SamplerConfig, sample_game
    import signal
    out = []
    for i in range(tries):
        if len(out) >= limit:
            break
        text = sample_game(SamplerConfig(seed=sampler_seed, max_depth=depth), index=i)
        try:
            signal.alarm(10)
            g = boardlang.load_game(text)
            runs = []
            for seed in (1, 2):
                po = engine.playout_random(g, seed=seed, batch_size=16, max_turns=60)
                runs.append({"seed": seed, "digest": po.final.digest(),
                             "turns": int(po.turns_taken.sum())})
            signal.alarm(0)
        except Exception:
            signal.alarm(0)
            continue
        out.append({"sampler": [sampler_seed, depth], "index": i, "text": text, "runs": runs})
    return out


def gavel_fixtures(n_valid=10, n_invalid=4):
    """GAVEL reports (evaluation.evaluate_game) of generated programs: valid
    ones (playable or stuck) and a few invalid ones, small match config."""
    from boardlang.evaluation import EvalConfig, evaluate_game
    from boardlang.generator import SamplerConfig, sample_game
    from boardlang.topology import build_topology
    from boardlang.validate import validate
    cfg = {"matches": 4, "strong_iterations": 8, "weak_iterations": 4, "max_turns": 60, "seed": 3}
    out, nv, ni = [], 0, 0
    for i in range(2000):
        if nv >= n_valid and ni >= n_invalid:
            break
        text = sample_game(SamplerConfig(seed=11, max_depth=6), index=i)
        spec = parse_game(text)
        ok = validate(spec, build_topology(spec.equipment.board)).ok
        if (ok and nv >= n_valid) or (not ok and ni >= n_invalid):
            continue
        rep = evaluate_game(text, EvalConfig(**cfg)).as_dict()
        if ok:
            nv += 1
        else:
            ni += 1
        out.append({"index": i, "text": text, "report": {k: (float.hex(v) if isinstance(v, float)
                                                            else v) for k, v in rep.items()}})
        print("gavel", i, rep.get("playable"), rep.get("diagnostic", "")[:60])
    with open(os.path.join(OUT, "gavel.json"), "w") as fh:
        json.dump({"config": cfg, "programs": out}, fh, indent=0, sort_keys=True)


def fuzz_mask_fixtures(stride=10):
    """Per-ply legal-mask hashes and sampled actions of B=4 trajectories
    (seed 3, 60-ply cap) for every `stride`-th fuzz program: exercises the
    mask writers and verified steps, not just final states."""
    import hashlib
    from boardlang import rng as rrng
    with open(os.path.join(OUT, "fuzz.json")) as fh:
        progs = json.load(fh)["programs"][::stride]
    out = []
    for prog in progs:
        g = boardlang.load_game(prog["text"])
        st = g.init(batch_size=4, seed=3)
        rows = [[] for _ in range(4)]
        for _ in range(60):
            if st.terminated.all():
                break
            m = g.legal_mask(st)
            u = rrng.uniform(st.seeds, st.move_count.astype(np.uint64))
            a = g.sample_actions(st, u)
            live = ~st.terminated
            if (a[live] < 0).any():
                break
            for i in np.nonzero(live)[0]:
                h = hashlib.blake2b(np.packbits(m[i]).tobytes(), digest_size=8).hexdigest()
                rows[i].append([h, int(a[i])])
            g.step_into(st, a, rows=live, verify=True)
        out.append({"sampler": prog.get("sampler"), "index": prog["index"], "rows": rows,
                    "digest": st.digest()})
    with open(os.path.join(OUT, "fuzz_masks.json"), "w") as fh:
        json.dump({"stride": stride, "programs": out}, fh, indent=0, sort_keys=True)
    print("wrote fuzz_masks.json", len(out))


def validate_fixtures(per_corpus=150):
    """Validation reports of generated programs, valid or not (validate.py,
    raised as ValidationFailure by load_game)."""
    from boardlang.generator import SamplerConfig, sample_game
    from boardlang.topology import build_topology
    from boardlang.validate import validate
    out = []
    for seed, depth in ((7, 5), (11, 6), (23, 8), (31, 10)):
        for i in range(per_corpus):
            text = sample_game(SamplerConfig(seed=seed, max_depth=depth), index=i)
            try:
                spec = parse_game(text)
                rep = str(validate(spec, build_topology(spec.equipment.board)))
            except Exception as exc:
                rep = f"EXC {type(exc).__name__}: {exc}"
            out.append({"sampler": [seed, depth], "index": i, "text": text, "report": rep})
    with open(os.path.join(OUT, "validate.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print("wrote validate.json", len(out), sum(o["report"] == "valid" for o in out), "valid")


def mover_fixtures(B=24, plies=(0, 3, 7, 15)):
    """Legality for a non-current mover (CompiledGame.legal_mask / legal_counts
    / sample_actions with mover=, compiler.py:394-446) on reference states of
    every corpus game: the states after k uniform-random plies, the mover
    flipped (and, for half the rows, kept), the reference's answers."""
    arrays = {}
    for name in GAMES:
        g = boardlang.load_game(open(os.path.join(GAMES_DIR, f"{name}.ldx")).read())
        st = g.init(batch_size=B, seed=4242)
        done = 0
        for k in range(max(plies) + 1):
            if k in plies:
                mover = (1 - st.current_player).astype(np.int8)
                mover[::2] = st.current_player[::2]
                u = rng.uniform(st.seeds, st.move_count.astype(np.uint64))
                pre = f"{name}__{k}__"
                arrays.update({k: v.copy() for k, v in state_arrays(st, pre).items()})
                arrays[pre + "mover"] = mover
                arrays[pre + "u"] = u
                arrays[pre + "mask"] = g.legal_mask(st, mover=mover)
                arrays[pre + "counts"] = g.legal_counts(st, mover=mover)
                arrays[pre + "sampled"] = g.sample_actions(st, u, mover=mover)
                done += 1
            live = ~st.terminated
            if not live.any():
                break
            acts = engine.random_actions(g, st)
            g.step_into(st, np.where(acts < 0, 0, acts), rows=live & (acts >= 0), verify=False)
        print("mover fixtures", name, done)
    np.savez_compressed(os.path.join(OUT, "mover.npz"), **arrays)


def program_fixtures():
    """Reference playouts of the test programs in tests/programs/ (not corpus
    games: programs that pin one property each, e.g. big_score.ldx's scores
    beyond int16): final-state digests, scores and outcomes."""
    pdir = os.path.join(os.path.dirname(OUT), "programs")
    out = {}
    for fn in sorted(os.listdir(pdir)):
        if not fn.endswith(".ldx"):
            continue
        g = boardlang.load_game(open(os.path.join(pdir, fn)).read())
        runs = []
        for B, seed in ((64, 3), (256, 11)):
            f = engine.playout_random(g, seed=seed, batch_size=B, max_turns=200).final
            runs.append({"batch": B, "seed": seed, "digest": f.digest(),
                         "scores": f.scores.tolist() if f.scores is not None else None,
                         "outcome": f.outcome.tolist(), "move_count": f.move_count.tolist()})
        out[fn[:-4]] = runs
    with open(os.path.join(OUT, "programs.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print("wrote programs.json", sorted(out))


if __name__ == "__main__":
    if "--programs" in sys.argv:
        program_fixtures()
        sys.exit(0)
    if "--mover" in sys.argv:
        mover_fixtures()
        sys.exit(0)
    if "--fuzz-masks" in sys.argv:
        fuzz_mask_fixtures()
        sys.exit(0)
    if "--gavel" in sys.argv:
        gavel_fixtures()
        sys.exit(0)
    if "--validate" in sys.argv:
        validate_fixtures()
        sys.exit(0)
    if "--fuzz" in sys.argv:
        fuzz_fixtures()
        sys.exit(0)
    if "--mcts" in sys.argv:
        mcts_fixtures()
    elif "--jsonl" in sys.argv:
        jsonl_fixtures()
    else:
        main()
        mcts_fixtures()
        jsonl_fixtures()
