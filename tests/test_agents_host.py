"""Host-side agent / GAVEL logic against the reference's own numbers
(tests/golden/mcts.json): score_match and harmonic_mean on the reference's
recorded match statistics, masked_choice / random_action draws."""
import json
import os

import numpy as np

from conftest import GOLDEN
from paper_2506_22609_b200 import agents, evaluation, rng

with open(os.path.join(GOLDEN, "mcts.json")) as f:
    MCTS = json.load(f)


def match_stats(d):
    st = agents.MatchStats(games=d["games"])
    for k in ("wins_p1", "wins_p2", "draws", "truncations", "multi_choice_turns",
              "total_turns", "wins_a", "wins_b"):
        setattr(st, k, d[k])
    st.turns = np.array(d["turns"])
    st.legal_counts = np.array(d["legal_counts"])
    st.coverage = np.array([float.fromhex(x) for x in d["coverage"]])
    st.seat_of_a = np.array(d["seat_of_a"], dtype=np.int8)
    st.winner_agent = np.array(d["winner_agent"], dtype=np.int8)
    return st


def test_score_match_matches_reference():
    for m in MCTS["matches"]:
        st = match_stats(m["stats"])
        st.check()
        sc = evaluation.score_match(st)
        assert {k: float.hex(v) for k, v in sc.as_dict().items()} == m["scores"], m["game"]
        assert float.hex(evaluation.harmonic_mean(sc.values())) == m["gavel"]


def test_random_action_and_masked_choice():
    mask = np.zeros(9, dtype=bool)
    mask[[1, 4, 7]] = True
    picks = {agents.random_action(mask, seed=3, counter=c) for c in range(64)}
    assert picks == {1, 4, 7}
    u = np.array([0.0, 0.999999, 0.5])
    m = np.array([[1, 0, 1], [1, 1, 1], [0, 0, 0]], dtype=bool)
    assert rng.masked_choice(m, u).tolist() == [0, 2, -1]


def test_gavel_csv_columns():
    rep = evaluation.GavelReport(name="x", playable=True,
                                 scores=evaluation.HeuristicScores(balance=0.5))
    csv = evaluation.gavel_csv([rep])
    assert csv.splitlines()[0] == ",".join(evaluation.GAVEL_CSV_COLUMNS)
    assert csv.splitlines()[1].startswith("x,True,0.5,")
