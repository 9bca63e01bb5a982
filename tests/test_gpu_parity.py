"""Device path vs the CPU oracle and the reference's golden fixtures.

Bit-exact comparisons on the reference GameState layout (digest = the
reference's own blake2b over every field).  All tests call through the
C-ABI (libludax_b200.so) via the package API.
"""
import numpy as np
import pytest

from conftest import GAMES, golden_arrays, golden_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402
from oracle import oracle as O  # noqa: E402

_GAMES = {}


def game(name):
    if name not in _GAMES:
        _GAMES[name] = lx.load_config_game(name)
    return _GAMES[name]


ORACLE_B = {"tic_tac_toe": 65536, "connect_four": 16384, "hex": 2048, "reversi": 4096,
            "pente": 512, "gomoku": 1024, "yavalath": 8192, "english_draughts": 4096,
            "dai_hasami_shogi": 1024, "wolf_and_sheep": 8192, "gridworld": 65536}


@pytest.mark.parametrize("name", GAMES)
def test_playout_matches_reference_fixtures(name, golden_meta):
    g = game(name)
    for k, p in enumerate(golden_meta["games"][name]["playouts"]):
        final = lx.engine.playout_random(g, seed=p["seed"], batch_size=p["batch"]).final
        want = golden_state(name, k)
        host = final.host()
        for f, v in want.items():
            assert np.array_equal(host[f], v), (name, k, f)
        assert final.digest() == p["digest"]


@pytest.mark.parametrize("name", GAMES)
def test_playout_matches_oracle_large(name):
    B = ORACLE_B[name]
    final = lx.engine.playout_random(game(name), seed=2024, batch_size=B).final
    want, _ = O.OracleGame(name).playout(B, seed=2024, threads=8)
    host = final.host()
    for f, v in want.items():
        assert np.array_equal(host[f], v), (name, f)


@pytest.mark.parametrize("name", GAMES)
def test_trajectory_masks_actions_digests(name, golden_meta):
    g = game(name)
    info = golden_meta["games"][name]
    arr = golden_arrays(name)
    width = info["traj_mask_width"]
    masks = np.unpackbits(arr["traj_masks"], axis=-1)[..., :width].astype(bool)
    st = g.init(batch_size=4, seed=3)
    for t in range(len(arr["traj_actions"])):
        assert np.array_equal(g.legal_mask(st), masks[t]), (name, t)
        a = lx.engine.random_actions(g, st)
        assert np.array_equal(a, arr["traj_actions"][t]), (name, t)
        g.step_into(st, a, rows=~st.terminated, verify=False)
        assert st.digest() == info["traj_digests"][t], (name, t)


@pytest.mark.parametrize("name", GAMES)
def test_replay_oracle_actions_stepwise(name):
    """Recorded-trajectory replay: step both sides with the same actions and
    compare every field after every ply, plus legal masks and counts."""
    g, og = game(name), O.OracleGame(name)
    B = 257
    st = g.init(batch_size=B, seed=99)
    ost = og.init(B, seed=99)
    for ply in range(210):
        m, cnt = og.legal_mask(ost)
        assert np.array_equal(g.legal_mask(st), m), (name, ply)
        assert np.array_equal(g.legal_counts(st), cnt), (name, ply)
        if ost["terminated"].all():
            break
        a = og.sample_actions(ost)
        live = ~ost["terminated"]
        og.step_into(ost, a, rows=live, verify=False)
        g.step_into(st, a, rows=live, verify=False)
        assert st.digest() == O.digest(ost), (name, ply)


@pytest.mark.parametrize("name", GAMES)
def test_export_import_roundtrip(name):
    og = O.OracleGame(name)
    ost = og.init(300, seed=5)
    for _ in range(9):
        a = og.sample_actions(ost)
        og.step_into(ost, a, rows=~ost["terminated"], verify=False)
    st = game(name).from_reference(ost)
    assert st.digest() == O.digest(ost)
    # and it keeps playing identically from the imported position
    lx.engine.playout_random(game(name), state=st)  # pure: st unchanged
    fin = lx.engine.playout_random(game(name), state=st).final
    want, _ = og.playout(state=ost)
    assert fin.digest() == O.digest(want)


def test_sample_with_host_uniforms():
    g, og = game("reversi"), O.OracleGame("reversi")
    st, ost = g.init(512, seed=1), og.init(512, seed=1)
    u = np.random.default_rng(0).random(512)
    assert np.array_equal(g.sample_actions(st, u), og.sample_actions(ost, u))


def test_known_answers(golden_meta):
    kat = golden_meta["kat"]
    ttt = game("tic_tac_toe")
    s = ttt.init(1)
    for a in kat["ttt_diag"]["actions"]:
        s = lx.engine.step(ttt, s, a)
    assert s.digest() == kat["ttt_diag"]["digest"]
    assert lx.engine.outcome_view(s) == {"p1": "win", "p2": "lose", "truncated": False}
    c4 = game("connect_four")
    assert np.nonzero(lx.engine.legal_actions(c4, c4.init(1))[0])[0].tolist() == \
        kat["c4_initial_legal"]
    rv = game("reversi")
    assert np.nonzero(lx.engine.legal_actions(rv, rv.init(1))[0])[0].tolist() == \
        kat["reversi_initial_legal"]
    pe = game("pente")
    for key in ("pente_capture", "pente_no_capture3"):
        s = pe.init(1)
        for a in kat[key]["actions"]:
            s = pe.step(s, np.array([a]))
        assert s.board_owner[0].tolist() == kat[key]["owner"]
        assert s.digest() == kat[key]["digest"]


def test_errors_map_to_reference_types():
    ttt = game("tic_tac_toe")
    s = lx.engine.step(ttt, ttt.init(1), 4)
    with pytest.raises(lx.IllegalAction):
        lx.engine.step(ttt, s, 4)
    for a in (0, 1, 2, 8):
        s = lx.engine.step(ttt, s, a) if not s.terminated[0] else s
    s = ttt.init(1)
    for a in [0, 1, 4, 2, 8]:
        s = lx.engine.step(ttt, s, a)
    with pytest.raises(lx.TerminalState):
        lx.engine.step(ttt, s, 3)
    with pytest.raises(lx.TerminalState):
        lx.engine.legal_actions(ttt, s)
    rv = game("reversi")
    with pytest.raises(lx.IllegalAction):       # pass is illegal while moves exist
        rv.step(rv.init(1), np.array([64]))


def test_step_is_pure():
    g = game("connect_four")
    s = g.init(2, seed=1)
    d0 = s.digest()
    s1 = g.step(s, np.array([35, 41]))
    s2 = g.step(s, np.array([35, 41]))
    assert s1.digest() == s2.digest() and s.digest() == d0


def test_batch_equals_sequential_and_partition():
    for name in GAMES:
        g = game(name)
        seeds = lx.rng.spawn_seeds(1234, 8)
        whole = lx.engine.playout_random(g, state=g.init(8, seeds=seeds)).final
        singles = [lx.engine.playout_random(g, state=g.init(1, seeds=seeds[i:i + 1])).final
                   for i in range(8)]
        assert whole.digest() == lx.DeviceState.concat(singles).digest(), name
        # shard by first_index: two halves == one batch (multi-GPU partition)
        left, _ = g.rollout(batch_size=512, seed=77)
        right, _ = g.rollout(batch_size=512, seed=77, first_index=512)
        full, _ = g.rollout(batch_size=1024, seed=77)
        assert lx.DeviceState.concat([left, right]).digest() == full.digest(), name


def test_record_mode_matches_fused(golden_meta):
    for name in GAMES:
        g = game(name)
        a = lx.engine.playout_random(g, seed=3, batch_size=16, record=True)
        b = lx.engine.playout_random(g, seed=3, batch_size=16)
        assert a.final.digest() == b.final.digest(), name
        rows = a.trajectory(0)
        assert rows[0]["move_count"] == 0 and rows[-1]["terminated"]


def test_truncation_marks_draw():
    g = game("pente")
    f = lx.engine.playout_random(g, seed=5, batch_size=64, max_turns=40).final
    tr = f.truncated
    assert tr.any() and (f.outcome[tr] == 0).all() and (f.move_count[tr] == 40).all()
    want, _ = O.OracleGame("pente").playout(64, seed=5, max_turns=40)
    assert f.digest() == O.digest(want)


def test_hex_no_draws_10000():
    f = lx.engine.playout_random(game("hex"), seed=404, batch_size=10_000).final
    assert f.terminated.all() and not f.truncated.any() and (f.outcome != 0).all()


def test_reversi_integrity_1000():
    f = lx.engine.playout_random(game("reversi"), seed=777, batch_size=1000).final
    p1 = (f.board_owner == 0).sum(axis=1)
    p2 = (f.board_owner == 1).sum(axis=1)
    assert (f.scores.sum(axis=1) == p1 + p2).all()
    assert (f.outcome == np.where(p1 > p2, 1, np.where(p2 > p1, 2, 0))).all()


def test_c4_opening_distribution(golden_meta):
    g = game("connect_four")
    st = g.init(batch_size=100_000, seed=77)
    a = lx.engine.random_actions(g, st)
    vals, cnt = np.unique(a, return_counts=True)
    assert dict(zip(map(str, vals.tolist()), cnt.tolist())) == golden_meta["kat"]["c4_opening_counts"]


def test_ttt_outcome_counts(golden_meta):
    want = golden_meta["kat"]["ttt_10000_seed11"]
    f = lx.engine.playout_random(game("tic_tac_toe"), seed=11, batch_size=10_000).final
    assert f.digest() == want["digest"]


def test_ttt_exhaustive_census():
    """Every tic-tac-toe game by breadth-first expansion on the device
    (reference test_acceptance.py:84-111): the published census 255168 games,
    131184 P1 wins, 77904 P2 wins, 46080 draws."""
    g = game("tic_tac_toe")
    st = g.init(1, seed=0)
    totals = np.zeros(4, dtype=np.int64)
    while st.batch_size:
        mask = g.legal_mask(st)
        counts = mask.sum(axis=1)
        rows, acts = np.nonzero(mask)
        st = st.rows(rows)
        g.step_into(st, acts.astype(np.int64), verify=False)
        m = g.meta(st)
        done = m["terminated"]
        totals += [done.sum(), (m["outcome"][done] == 1).sum(), (m["outcome"][done] == 2).sum(),
                   (m["outcome"][done] == 0).sum()]
        st = st.rows(np.nonzero(~done)[0]) if (~done).any() else st.rows([])
    assert tuple(int(x) for x in totals) == (255168, 131184, 77904, 46080)


def test_connect_four_opening_chi_square():
    """1e5 uniform openings (reference test_agents.py:28-41)."""
    g = game("connect_four")
    n = 100_000
    a = lx.engine.random_actions(g, g.init(n, seed=77))
    vals, cnt = np.unique(a, return_counts=True)
    assert vals.tolist() == list(range(35, 42))
    exp = n / 7
    assert float(((cnt - exp) ** 2 / exp).sum()) < 22.46


def test_hex_cooperative_flood_matches_per_lane_flood(monkeypatch):
    """Hex reach sets grown by the warp-cooperative flood (lx::coop_flood,
    full warps) and by the per-lane flood (LX_COOP_FLOOD=0 lowering) give
    identical final states at full size, and both match the oracle on a
    sample; partial warps (odd batch) take the per-lane path."""
    import os
    path = os.path.join(lx.game.GAMES_DIR, "hex.ldx")
    with open(path) as f:
        text = f.read()
    coop = lx.load_game(text)
    monkeypatch.setenv("LX_COOP_FLOOD", "0")
    solo = lx.load_game(text)
    assert coop.lowered_key() != solo.lowered_key()
    for B, seed in ((1 << 18, 3), (1000, 11)):
        a = lx.engine.playout_random(coop, seed=seed, batch_size=B).final.digest()
        b = lx.engine.playout_random(solo, seed=seed, batch_size=B).final.digest()
        assert a == b, (B, seed)
    want, _ = O.OracleGame("hex").playout(1000, seed=11)
    assert a == O.digest(want)


# full BASELINE size (2^22 envs per GPU) for every corpus game: the fused
# rollout's per-env outcome and ply count, spot-checked window by window
# against the oracle replaying the same env indices (seeds = spawn(seed, i),
# reference rng.py:45-54) -- head, a seeded interior window and the tail
FULL_B = 1 << 22
SPOT_W = {"tic_tac_toe": 16384, "connect_four": 8192, "hex": 2048, "reversi": 2048,
          "pente": 1024, "gomoku": 1024, "yavalath": 2048, "english_draughts": 1024,
          "dai_hasami_shogi": 512, "wolf_and_sheep": 2048, "gridworld": 16384}


@pytest.mark.parametrize("name", list(SPOT_W))
def test_full_size_rollout_windows_match_oracle(name):
    g = game(name)
    W = SPOT_W[name]
    out = torch.empty(FULL_B, dtype=torch.int8, device="cuda")
    turns = torch.empty(FULL_B, dtype=torch.int32, device="cuda")
    _, st = g.rollout(batch_size=FULL_B, seed=4242, store=False, outcomes=out, turns=turns)
    st = st.cpu().tolist()
    assert st[5] == FULL_B and st[1] + st[2] + st[3] == FULL_B
    mid = int(np.random.default_rng(7).integers(W, FULL_B - 2 * W))
    og = O.OracleGame(name)
    for off in (0, mid, FULL_B - W):
        want, _ = og.playout(seeds=O.spawn_seeds(4242, W, first=off), threads=8)
        got_o = out[off:off + W].cpu().numpy()
        got_t = turns[off:off + W].cpu().numpy()
        assert np.array_equal(got_o, want["outcome"]), (name, off)
        assert np.array_equal(got_t, want["move_count"]), (name, off)
