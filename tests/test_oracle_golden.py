"""The CPU oracle is pinned to fixtures produced by the reference itself."""
import numpy as np
import pytest

from conftest import GAMES, golden_arrays, golden_state
from oracle import oracle as O


@pytest.mark.parametrize("name", GAMES)
def test_oracle_playouts_match_reference(name, golden_meta):
    og = O.OracleGame(name)
    for k, p in enumerate(golden_meta["games"][name]["playouts"]):
        st, steps = og.playout(p["batch"], seed=p["seed"])
        want = golden_state(name, k)
        for f, v in want.items():
            assert np.array_equal(st[f], v), (name, k, f)
        assert O.digest(st) == p["digest"]
        assert int(st["move_count"].sum()) == p["turns"]


@pytest.mark.parametrize("name", GAMES)
def test_oracle_trajectory_masks_and_actions(name, golden_meta):
    og = O.OracleGame(name)
    info = golden_meta["games"][name]
    arr = golden_arrays(name)
    width = info["traj_mask_width"]
    masks = np.unpackbits(arr["traj_masks"], axis=-1)[..., :width].astype(bool)
    st = og.init(batch_size=4, seed=3)
    for t in range(len(arr["traj_actions"])):
        m, _ = og.legal_mask(st)
        assert np.array_equal(m, masks[t]), (name, t)
        a = og.sample_actions(st)
        assert np.array_equal(a, arr["traj_actions"][t]), (name, t)
        og.step_into(st, a, rows=~st["terminated"], verify=False)
        assert O.digest(st) == info["traj_digests"][t], (name, t)


def test_oracle_known_answers(golden_meta):
    kat = golden_meta["kat"]
    ttt = O.OracleGame("tic_tac_toe")
    s = ttt.init(1)
    for a in kat["ttt_diag"]["actions"]:
        assert ttt.step_into(s, np.array([a]))[0] == 0
    assert O.digest(s) == kat["ttt_diag"]["digest"]
    c4 = O.OracleGame("connect_four")
    m, _ = c4.legal_mask(c4.init(1))
    assert np.nonzero(m[0])[0].tolist() == kat["c4_initial_legal"]
    rv = O.OracleGame("reversi")
    m, _ = rv.legal_mask(rv.init(1))
    assert np.nonzero(m[0])[0].tolist() == kat["reversi_initial_legal"]
    pe = O.OracleGame("pente")
    for key in ("pente_capture", "pente_no_capture3"):
        s = pe.init(1)
        for a in kat[key]["actions"]:
            assert pe.step_into(s, np.array([a]))[0] == 0
        assert s["board_owner"][0].tolist() == kat[key]["owner"]
        assert O.digest(s) == kat[key]["digest"]


def test_oracle_illegal_action_status():
    ttt = O.OracleGame("tic_tac_toe")
    s = ttt.init(1)
    assert ttt.step_into(s, np.array([4]))[0] == 0
    st, bad = ttt.step_into(s, np.array([4]))
    assert st == 1 and bad == 0


def test_oracle_rng_vectors(golden_meta):
    r = golden_meta["kat"]["rng"]
    seeds = O.spawn_seeds(12345, 16)
    assert [str(int(x)) for x in seeds] == r["spawn_12345_16"]
    for key, v in r["episode_keys"].items():
        b, e = map(int, key.split("_"))
        assert str(O.hash_key3(0, b, e)) == v


def test_oracle_ttt_outcome_counts(golden_meta):
    want = golden_meta["kat"]["ttt_10000_seed11"]
    st, _ = O.OracleGame("tic_tac_toe").playout(10_000, seed=11, threads=4)
    assert O.digest(st) == want["digest"]
    assert int((st["outcome"] == 1).sum()) == want["p1"]
    assert int((st["outcome"] == 0).sum()) == want["draw"]
