"""Edge cases and full-size properties of the device path (vs the oracle)."""
import numpy as np
import pytest

from conftest import GAMES

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402
from oracle import oracle as O  # noqa: E402

_G = {}


def game(name):
    if name not in _G:
        _G[name] = lx.load_config_game(name)
    return _G[name]


@pytest.mark.parametrize("name", GAMES)
@pytest.mark.parametrize("B", [1, 31, 33, 257, 1000])
def test_odd_batch_sizes(name, B):
    f = lx.engine.playout_random(game(name), seed=B, batch_size=B).final
    want, _ = O.OracleGame(name).playout(B, seed=B)
    assert f.digest() == O.digest(want)


@pytest.mark.parametrize("name", GAMES)
@pytest.mark.parametrize("max_turns", [1, 5, 37])
def test_truncation_caps(name, max_turns):
    f = lx.engine.playout_random(game(name), seed=9, batch_size=300, max_turns=max_turns).final
    want, _ = O.OracleGame(name).playout(300, seed=9, max_turns=max_turns)
    assert f.digest() == O.digest(want)


@pytest.mark.parametrize("name", GAMES)
def test_explicit_extreme_seeds(name):
    rs = np.random.default_rng(1)
    seeds = np.concatenate([np.array([0, 1, 2**64 - 1, 2**63], dtype=np.uint64),
                            rs.integers(0, 2**63, 252, dtype=np.uint64) * 2 + 1])
    g, og = game(name), O.OracleGame(name)
    f = lx.engine.playout_random(g, state=g.init(len(seeds), seeds=seeds)).final
    want, _ = og.playout(state=og.init(len(seeds), seeds=seeds))
    assert f.digest() == O.digest(want)


@pytest.mark.parametrize("name", GAMES)
def test_partial_rows_and_terminal_outputs(name):
    g, og = game(name), O.OracleGame(name)
    B = 129
    st, ost = g.init(B, seed=4), og.init(B, seed=4)
    rs = np.random.default_rng(2)
    for ply in range(150):
        rows = rs.random(B) < 0.6
        a = og.sample_actions(ost)
        og.step_into(ost, a, rows=rows, verify=False)
        g.step_into(st, a, rows=rows, verify=False)
        if ply % 10 == 0:
            assert st.digest() == O.digest(ost), ply
    m, cnt = og.legal_mask(ost)
    term = ost["terminated"]
    assert np.array_equal(g.legal_mask(st), m) and np.array_equal(g.legal_counts(st), cnt)
    assert not g.legal_mask(st)[term].any() and (g.legal_counts(st)[term] == 0).all()
    acts = g.sample_actions(st, np.full(B, 0.5))
    assert (acts[term] == -1).all()


@pytest.mark.parametrize("name", GAMES)
def test_verify_reports_first_illegal_row(name):
    g, og = game(name), O.OracleGame(name)
    st, ost = g.init(64, seed=8), og.init(64, seed=8)
    for _ in range(6):
        a = og.sample_actions(ost)
        og.step_into(ost, a, verify=False)
        g.step_into(st, a, verify=False)
    m, _ = og.legal_mask(ost)
    a = og.sample_actions(ost)
    live = np.nonzero(~ost["terminated"])[0]
    bad_rows = live[[5, 9]] if len(live) > 9 else live[:1]
    for r in bad_rows:
        illegal = np.nonzero(~m[r])[0]
        a[r] = illegal[0] if len(illegal) else -7
    before = st.digest()
    with pytest.raises(lx.IllegalAction) as e:
        g.step_into(st, a, verify=True)
    assert f"row {bad_rows[0]}" in str(e.value)
    assert st.digest() == before          # nothing was applied


def test_reversi_pass_only_states_and_pass_step():
    g, og = game("reversi"), O.OracleGame("reversi")
    st, ost = g.init(512, seed=3), og.init(512, seed=3)
    seen = 0
    for _ in range(70):
        m, cnt = og.legal_mask(ost)
        dm = g.legal_mask(st)
        assert np.array_equal(dm, m)
        pass_only = ~ost["terminated"] & m[:, 64] & (cnt == 1)
        seen += int(pass_only.sum())
        a = og.sample_actions(ost)
        og.step_into(ost, a, verify=True)
        g.step_into(st, a, verify=True)
    assert seen > 0 and st.digest() == O.digest(ost)


def test_auto_reset_matches_reference_semantics():
    g, og = game("tic_tac_toe"), O.OracleGame("tic_tac_toe")
    st, ost = g.init(64, seed=1), og.init(64, seed=1)
    for _ in range(15):
        a = og.sample_actions(ost)
        a = np.where(a < 0, 0, a)
        st = lx.engine.step_batch(g, st, a, auto_reset=True)
        og.step_into(ost, a, verify=False)
        done = ost["terminated"]
        if done.any():                 # engine.reset_rows (engine.py:58-65)
            idx = np.nonzero(done)[0]
            fresh = og.init(len(idx), seeds=lx.rng.hash_key(ost["seeds"][idx], np.uint64(0xE9)))
            for k, v in fresh.items():
                ost[k][idx] = v
        assert st.digest() == O.digest(ost)


@pytest.mark.parametrize("name", GAMES)
def test_observe_planes(name):
    g = game(name)
    st = lx.engine.playout_random(g, seed=2, batch_size=64, max_turns=7).final
    own, pc = st.board_owner, st.board_piece
    T = len(g.piece_names)
    for p in (0, 1):
        planes, mask = g.observe(st, p)
        assert planes.shape[1] == 2 * T + 1
        for t in range(T):
            assert np.array_equal(planes[:, 2 * t], (own == p) & (pc == t))
            assert np.array_equal(planes[:, 2 * t + 1], (own == 1 - p) & (pc == t))
        assert np.array_equal(planes[:, 2 * T], np.repeat((st.current_player == p)[:, None],
                                                           g.num_cells, axis=1))
        assert np.array_equal(mask, g.legal_mask(st))


def test_full_size_c4_properties_and_shards():
    """2^22 envs: stat identities, determinism, and 4 shards == one batch."""
    g = game("connect_four")
    B = 1 << 22
    out = torch.empty(B, dtype=torch.int8, device="cuda")
    turns = torch.empty(B, dtype=torch.int32, device="cuda")
    _, s1 = g.rollout(batch_size=B, seed=5, store=False, outcomes=out, turns=turns)
    s1 = s1.cpu().tolist()
    assert s1[1] + s1[2] + s1[3] == s1[5] == B
    assert s1[0] == int(turns.sum().item())
    assert int((out == 1).sum()) == s1[1] and int((out == 0).sum()) == s1[3]
    _, s2 = g.rollout(batch_size=B, seed=5, store=False)
    assert s2.cpu().tolist() == s1
    parts = []
    acc = np.zeros(8, dtype=np.int64)
    for k in range(4):
        o = torch.empty(B // 4, dtype=torch.int8, device="cuda")
        _, s = g.rollout(batch_size=B // 4, seed=5, store=False, first_index=k * (B // 4),
                         outcomes=o)
        acc += s.cpu().numpy()
        parts.append(o)
    assert acc[:6].tolist() == s1[:6]             # [6] is the stuck row (~0 = none), not a count
    assert torch.equal(torch.cat(parts), out)


def test_full_size_hex_no_draws_and_reversi_conservation():
    _, s = game("hex").rollout(batch_size=1 << 20, seed=11, store=False)
    s = s.cpu().tolist()
    assert s[3] == 0 and s[4] == 0 and s[1] + s[2] == 1 << 20
    f, _ = game("reversi").rollout(batch_size=1 << 18, seed=12)
    h = f.host()
    p1 = (h["board_owner"] == 0).sum(axis=1)
    p2 = (h["board_owner"] == 1).sum(axis=1)
    assert (h["scores"][:, 0] == p1).all() and (h["scores"][:, 1] == p2).all()
    assert (h["outcome"] == np.where(p1 > p2, 1, np.where(p2 > p1, 2, 0))).all()


@pytest.mark.parametrize("name", GAMES)
def test_mcts_rollout_primitive(name):
    """engine.rollout_outcomes == reference agents._rollout semantics: continue
    from mid-game states with re-keyed seeds (agents.py:229-233), draws at the cap."""
    g, og = game(name), O.OracleGame(name)
    B = 200
    st, ost = g.init(B, seed=21), og.init(B, seed=21)
    for _ in range(5):
        a = og.sample_actions(ost)
        og.step_into(ost, a, verify=False)
        g.step_into(st, a, verify=False)
    keys = lx.rng.hash_key(np.uint64(777), np.uint64(0x5011), np.arange(B, dtype=np.uint64))
    got = lx.engine.rollout_outcomes(g, st, max_turns=60, seeds=keys).cpu().numpy()
    ost["seeds"][:] = keys
    fin, _ = og.playout(state=ost, max_turns=60)
    want = np.where(fin["terminated"] & ~fin["truncated"], fin["outcome"], 0)
    assert np.array_equal(got, want)
    assert st.digest() != O.digest(fin)        # input state untouched (still mid-game)


def test_host_edits_of_exported_fields_reach_the_device():
    """DeviceState write-back: in-place edits of exported reference
    fields -- what engine.playout_random does at the cap (engine.py:156-160)
    -- are imported before the next device call, so the device sees them."""
    g = game("connect_four")
    st = g.init(4, seed=1)
    st.terminated[1] = True                      # host-side edits of the cached export
    st.truncated[1] = True
    st.outcome[1] = 0
    g.step_into(st, np.array([35, 36, 37, 38]), verify=False)
    assert st.move_count.tolist() == [1, 0, 1, 1]          # row 1 absorbed the step
    assert st.terminated.tolist() == [False, True, False, False]
    assert bool(st.truncated[1]) and int(st.outcome[1]) == 0
    cp = st.copy()                                # copies see the edits too
    cp.outcome[2] = 1
    cp.terminated[2] = True
    fin, _ = g.rollout(state=cp, max_turns=200)
    assert int(fin.outcome[2]) == 1 and int(fin.move_count[2]) == 1


def test_rollout_work_buffer_is_left_clear_and_clear_mode():
    """lx_rollout needs no memsets: the last block publishes the stats and
    leaves the 128-byte work buffer zeroed; LX_ROLLOUT_CLEAR_WORK (mode bit 3)
    clears a buffer the caller cannot vouch for."""
    import ctypes

    from paper_2506_22609_b200 import native
    g = game("connect_four")
    B = 3000
    work = torch.zeros(16, dtype=torch.int64, device="cuda")
    _, s1 = g.rollout(batch_size=B, seed=9, store=False, work=work)
    assert int(work.abs().sum()) == 0
    want = s1.cpu().tolist()
    assert want[6] == -1                                     # no stuck row
    work.fill_(12345)                                        # dirty scratch
    stats = torch.empty(8, dtype=torch.int64, device="cuda")
    stuck = ctypes.c_int64(-1)
    native.check(native.lib().lx_rollout(g.handle, None, B, 200, 1 | 4 | 8, 9, None, 0,
                                         stats.data_ptr(), work.data_ptr(), None, None, 1,
                                         ctypes.byref(stuck), g._stream()))
    assert stats.cpu().tolist() == want and int(work.abs().sum()) == 0
