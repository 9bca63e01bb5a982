"""MCTS / match runner / GAVEL scoring and the JSONL trajectory format on the
device path against the reference's own outputs
(tests/golden/mcts.json, jsonl.json made by oracle/gen_golden.py)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, game_text

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402
from paper_2506_22609_b200 import agents, evaluation  # noqa: E402

with open(os.path.join(GOLDEN, "mcts.json")) as f:
    MCTS = json.load(f)
with open(os.path.join(GOLDEN, "jsonl.json")) as f:
    JSONL = json.load(f)

_G = {}


def game(name):
    if name not in _G:
        _G[name] = lx.load_config_game(name)
    return _G[name]


def policy(p):
    if p[0] == "mcts":
        return agents.MctsPolicy(agents.MctsConfig(iterations=p[1], seed=p[2]))
    return agents.RandomPolicy(seed=p[1])


def stats_dict(st):
    return {"games": st.games, "wins_p1": st.wins_p1, "wins_p2": st.wins_p2, "draws": st.draws,
            "truncations": st.truncations, "turns": st.turns.tolist(),
            "legal_counts": st.legal_counts.tolist(),
            "multi_choice_turns": st.multi_choice_turns, "total_turns": st.total_turns,
            "coverage": [float.hex(float(x)) for x in st.coverage],
            "seat_of_a": st.seat_of_a.tolist(), "winner_agent": st.winner_agent.tolist(),
            "wins_a": st.wins_a, "wins_b": st.wins_b}


@pytest.mark.parametrize("m", MCTS["matches"], ids=lambda m: f"{m['game']}-{m['a'][0]}-{m['b'][0]}")
def test_play_match_matches_reference(m):
    st = agents.play_match(game(m["game"]), policy(m["a"]), policy(m["b"]), m["games"],
                           seed=m["seed"], max_turns=m["max_turns"])
    assert stats_dict(st) == m["stats"]


@pytest.mark.parametrize("s", MCTS["searches"], ids=lambda s: s["game"])
def test_mcts_search_matches_reference(s):
    g = game(s["game"])
    st = g.init(1, seed=s["init_seed"])
    for a in s["actions"]:
        st = g.step(st, np.array([a]))
    best = agents.mcts_search(g, st, agents.MctsConfig(iterations=s["iterations"],
                                                       seed=s["seed"]))
    assert best == s["best"]


def test_gavel_report_matches_reference():
    c = MCTS["gavel_ttt"]["config"]
    rep = evaluation.evaluate_game(game_text("tic_tac_toe"),
                                   evaluation.EvalConfig(**c))
    assert rep.as_dict() == MCTS["gavel_ttt"]["report"]
    bad = evaluation.evaluate_game("(game \"broken\"")
    assert not bad.playable and bad.diagnostic


def test_terminal_search_raises():
    g = game("tic_tac_toe")
    s = g.init(1)
    for a in (0, 1, 4, 2, 8):
        s = lx.engine.step(g, s, a)
    with pytest.raises(lx.TerminalState):
        agents.mcts_search(g, s)


@pytest.mark.parametrize("name", sorted(JSONL))
def test_jsonl_trajectories_match_reference(name):
    f = JSONL[name]
    po = lx.engine.playout_random(game(name), seed=f["seed"], batch_size=f["batch"], record=True)
    assert po.final.digest() == f["digest"]
    for i in range(f["batch"]):
        assert po.to_jsonl(i) == f["jsonl"][i]


def test_benchmark_throughput_report():
    g = game("connect_four")
    rep = evaluation.benchmark_throughput(g, [1024, 4096], warmup_episodes=2, episodes=3)
    assert rep.rate("Connect Four", 4096) > 0
    assert rep.to_csv().startswith("game,batch_size")


with open(os.path.join(GOLDEN, "gavel.json")) as f:
    GAVEL = json.load(f)


@pytest.mark.parametrize("prog", GAVEL["programs"], ids=lambda p: f"sample-{p['index']}")
def test_gavel_on_generated_programs(prog):
    """evaluate_game on programs from the reference's generator: same
    playable verdicts, diagnostics (ValidationFailure / EmptyMask /
    UnsupportedConstruct text) and scores as the reference."""
    rep = evaluation.evaluate_game(prog["text"], evaluation.EvalConfig(**GAVEL["config"]))
    got = {k: (float.hex(v) if isinstance(v, float) else v) for k, v in rep.as_dict().items()}
    assert got == prog["report"]


@pytest.mark.parametrize("name", ["connect_four", "reversi", "english_draughts", "hex"])
@pytest.mark.parametrize("shared", [True, False])
def test_device_search_equals_host_search(name, shared, monkeypatch):
    """lx_mcts (one warp per tree; the tree in shared memory, or in the
    global arena) and the host tree search make the same decisions on a
    batch of mid-game positions."""
    if not shared:
        monkeypatch.setattr(lx.game, "MCTS_SHARED_LIMIT", 0)
    g = game(name)
    st = g.init(12, seed=41)
    for _ in range(6):
        g.step_into(st, lx.engine.random_actions(g, st), rows=~st.terminated, verify=False)
    rows = ~st.terminated
    budgets = np.full(12, 24, dtype=np.int64)
    salt = np.full(12, np.uint64(9), dtype=np.uint64)
    search = agents._Search(g, 1.4142135623730951, 60)
    dev = search.run(st, rows, budgets, salt, device=True)
    host = search.run(st, rows, budgets, salt, device=False)
    assert np.array_equal(dev, host)


def test_device_search_shared_overflow_falls_back(monkeypatch):
    """A tree that passes the host's size check but does not fit beside the
    kernel's static shared buffers (lx_mcts returns LX_EINVALID) is searched
    in the global arena with the same decisions."""
    g = game("reversi")
    st = g.init(4, seed=3)
    rows = ~st.terminated
    budgets = np.full(4, 400, dtype=np.int64)        # ~245 KB of tree per root
    salt = np.full(4, np.uint64(5), dtype=np.uint64)
    search = agents._Search(g, 1.4142135623730951, 40)
    ref = search.run(st, rows, budgets, salt, device=True)
    monkeypatch.setattr(lx.game, "MCTS_SHARED_LIMIT", 1 << 30)   # skip the host check
    got = search.run(st, rows, budgets, salt, device=True)
    assert np.array_equal(got, ref)
    assert np.array_equal(got, search.run(st, rows, budgets, salt, device=False))


def test_device_search_on_generated_programs():
    """Device and host MCTS agree on programs from the reference's generator
    (movement, mixed phases, passes, transient masks ...)."""
    with open(os.path.join(GOLDEN, "fuzz.json")) as f:
        progs = json.load(f)["programs"][::57][:4]
    for prog in progs:
        g = lx.load_game(prog["text"])
        st = g.init(6, seed=5)
        for _ in range(3):
            live = ~st.terminated
            a = lx.engine.random_actions(g, st)
            if (a[live] < 0).any():
                break
            g.step_into(st, a, rows=live, verify=False)
        rows = ~st.terminated
        budgets = np.full(6, 12, dtype=np.int64)
        salt = np.full(6, np.uint64(3), dtype=np.uint64)
        search = agents._Search(g, 1.4142135623730951, 30)
        assert np.array_equal(search.run(st, rows, budgets, salt, device=True),
                              search.run(st, rows, budgets, salt, device=False)), prog["index"]
