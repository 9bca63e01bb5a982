"""Movement / gridworld games on the device against the
reference's own outputs: seeded playouts, per-ply masks / actions / digests,
the transcripts of the reference tests, and the engine / env surfaces.  All
calls go through the C-ABI (libludax_b200.so)."""
import numpy as np
import pytest

from conftest import MOVEMENT_GAMES, game_text, golden_arrays, golden_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402

_GAMES = {}


def game(name):
    if name not in _GAMES:
        _GAMES[name] = lx.load_config_game(name)
    return _GAMES[name]


@pytest.mark.parametrize("name", MOVEMENT_GAMES)
def test_movement_playout_matches_reference(name, golden_meta):
    g = game(name)
    for k, p in enumerate(golden_meta["games"][name]["playouts"]):
        po = lx.engine.playout_random(g, seed=p["seed"], batch_size=p["batch"])
        want = golden_state(name, k)
        host = po.final.host()
        assert set(host) == set(want), name
        for f, v in want.items():
            assert np.array_equal(host[f], v), (name, k, f)
        assert po.final.digest() == p["digest"]
        assert int(po.turns_taken.sum()) == p["turns"]


@pytest.mark.parametrize("name", MOVEMENT_GAMES)
def test_movement_trajectory(name, golden_meta):
    g = game(name)
    info = golden_meta["games"][name]
    arr = golden_arrays(name)
    width = info["traj_mask_width"]
    assert g.action_space_size == width
    masks = np.unpackbits(arr["traj_masks"], axis=-1)[..., :width].astype(bool)
    st = g.init(batch_size=4, seed=3)
    for t in range(len(arr["traj_actions"])):
        m = g.legal_mask(st)
        assert np.array_equal(m, masks[t]), (name, t)
        assert np.array_equal(g.legal_counts(st), m.sum(axis=1)), (name, t)
        a = lx.engine.random_actions(g, st)
        assert np.array_equal(a, arr["traj_actions"][t]), (name, t)
        g.step_into(st, a, rows=~st.terminated, verify=True)
        assert st.digest() == info["traj_digests"][t], (name, t)


def test_draughts_transcripts(golden_meta):
    kat = golden_meta["kat"]
    dr = game("english_draughts")
    s = dr.init(1)
    for a in kat["draughts_forced"]["actions"]:
        s = lx.engine.step(dr, s, a)
    assert np.nonzero(dr.legal_mask(s)[0])[0].tolist() == kat["draughts_forced"]["legal"]
    assert s.digest() == kat["draughts_forced"]["digest"]
    with pytest.raises(lx.IllegalAction):         # a step while a capture exists
        lx.engine.step(dr, s, 17 * 64 + 26)
    s = lx.engine.step(dr, s, 17 * 64 + 35)
    assert s.digest() == kat["draughts_forced"]["after_capture"]["digest"]
    assert int(s.current_player[0]) == 0
    drill = kat["draughts_drill"]
    text = game_text("english_draughts")
    for a, b in drill["text_replace"]:
        text = text.replace(a, b)
    g = lx.load_game(text)
    s = g.init(1)
    assert np.nonzero(g.legal_mask(s)[0])[0].tolist() == drill["start_legal"]
    s = g.step(s, np.array([36 * 64 + 18]))
    assert int(s.must_move[0]) == 18 and int(s.current_player[0]) == 0
    assert np.nonzero(g.legal_mask(s)[0])[0].tolist() == drill["after1"]["legal"]
    assert s.digest() == drill["after1"]["digest"]
    s = g.step(s, np.array([18 * 64 + 0]))
    assert int(s.board_piece[0, 0]) == 1 and int(s.current_player[0]) == 1
    assert s.digest() == drill["after2"]["digest"]


def test_gridworld_transcript(golden_meta):
    kat = golden_meta["kat"]["gridworld"]
    g = game("gridworld")
    assert list(g.codec.directions) == kat["directions"]
    s = g.init(1)
    assert np.nonzero(g.legal_mask(s)[0])[0].tolist() == kat["initial_legal"]
    for a in kat["right_down"]["actions"]:
        s = lx.engine.step(g, s, a)
    assert s.digest() == kat["right_down"]["digest"]
    assert lx.engine.outcome_view(s)["p1"] == "lose"


@pytest.mark.parametrize("name", MOVEMENT_GAMES)
def test_movement_batch_partition_record(name):
    g = game(name)
    seeds = lx.rng.spawn_seeds(1234, 8)
    whole = lx.engine.playout_random(g, state=g.init(8, seeds=seeds)).final
    singles = [lx.engine.playout_random(g, state=g.init(1, seeds=seeds[i:i + 1])).final
               for i in range(8)]
    assert whole.digest() == lx.DeviceState.concat(singles).digest()
    left, _ = g.rollout(batch_size=4096, seed=77)
    right, _ = g.rollout(batch_size=4096, seed=77, first_index=4096)
    full, _ = g.rollout(batch_size=8192, seed=77)
    assert lx.DeviceState.concat([left, right]).digest() == full.digest()
    a = lx.engine.playout_random(g, seed=3, batch_size=64, record=True)
    b = lx.engine.playout_random(g, seed=3, batch_size=64)
    assert a.final.digest() == b.final.digest()


@pytest.mark.parametrize("name", MOVEMENT_GAMES)
def test_movement_export_import_and_observe(name):
    g = game(name)
    st = g.init(300, seed=5)
    for _ in range(7):
        g.step_into(st, lx.engine.random_actions(g, st), rows=~st.terminated, verify=False)
    host = st.host()
    st2 = g.from_reference(host)
    assert st2.digest() == st.digest()
    fin = lx.engine.playout_random(g, state=st).final
    fin2 = lx.engine.playout_random(g, state=st2).final
    assert fin.digest() == fin2.digest()
    planes, mask = g.observe(st, 0)
    T = len(g.piece_names)
    assert planes.shape == (300, 2 * T + 1, g.num_cells)
    for t in range(T):
        assert np.array_equal(planes[:, 2 * t], (host["board_piece"] == t) & (host["board_owner"] == 0))
        assert np.array_equal(planes[:, 2 * t + 1], (host["board_piece"] == t) & (host["board_owner"] == 1))
    assert np.array_equal(planes[:, 2 * T], np.repeat((host["current_player"] == 0)[:, None],
                                                      g.num_cells, axis=1))
    assert np.array_equal(mask, g.legal_mask(st))


@pytest.mark.parametrize("name", MOVEMENT_GAMES)
def test_movement_env_step_masks(name):
    g = game(name)
    env = lx.LudaxEnvironment(g)
    es = env.init(batch_size=96, seed=4)
    for _ in range(30):
        m = es.legal_action_mask.cpu().numpy()
        assert np.array_equal(m, g.legal_mask(es.game_state))
        es = env.step(es, env.random_actions(es))


@pytest.mark.parametrize("name", MOVEMENT_GAMES)
def test_movement_large_batch_properties(name):
    g = game(name)
    B = 1 << 20
    fin, stats = g.rollout(batch_size=B, seed=11)
    st = stats.cpu().numpy()
    assert st[1] + st[2] + st[3] == B and st[5] == B
    out = fin.host()
    assert out["terminated"].all()
    assert ((out["outcome"] == 0) | ~out["truncated"]).all()
    # a random subset replayed in record mode (sample + step through the C-ABI)
    idx = np.random.default_rng(0).choice(B, 64, replace=False)
    seeds = lx.rng.spawn_seeds(11, B)[idx]
    sub = lx.engine.playout_random(g, state=g.init(64, seeds=seeds), record=True).final
    want = fin.rows(idx)
    assert sub.digest() == want.digest()
