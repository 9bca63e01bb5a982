"""PGX-style LudaxEnvironment on device vs the engine / oracle."""
import numpy as np
import pytest

from conftest import GAMES

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402
from oracle import oracle as O  # noqa: E402


@pytest.mark.parametrize("name", GAMES)
def test_env_random_episodes_match_playout(name):
    env = lx.LudaxEnvironment(name, max_steps=200)      # engine.playout_random's cap
    B = 512
    st = env.init(seed=42, batch_size=B)
    assert np.array_equal(st.legal_action_mask.cpu().numpy(),
                          env.game.legal_mask(st.game_state))
    assert not st.rewards.any() and not st.terminated.any()
    total = torch.zeros((B, 2), device="cuda")
    for _ in range(400):
        if bool(st.terminated.all()):
            break
        a = env.random_actions(st)
        st = env.step(st, a)
        total += st.rewards
        m = st.legal_action_mask.cpu().numpy()
        assert np.array_equal(m, env.game.legal_mask(st.game_state))
    want, _ = O.OracleGame(name).playout(B, seed=42, max_turns=200)
    host = st.game_state.host()
    for f in ("board_owner", "board_piece", "outcome", "move_count", "terminated", "truncated"):
        assert np.array_equal(host[f], want[f]), f
    out = want["outcome"]
    exp = np.stack([np.where(out == 1, 1.0, np.where(out == 2, -1.0, 0.0)),
                    np.where(out == 2, 1.0, np.where(out == 1, -1.0, 0.0))], axis=1)
    assert np.array_equal(total.cpu().numpy(), exp)


def test_env_step_is_functional_and_auto_reset():
    env = lx.LudaxEnvironment("tic_tac_toe", auto_reset=True)
    st = env.init(seed=1, batch_size=64)
    d0 = st.game_state.digest()
    st2 = env.step(st, env.random_actions(st))
    assert st.game_state.digest() == d0 and st2.game_state.digest() != d0
    done = 0
    for _ in range(40):
        prev_mc = st2.game_state.move_count.copy()
        st2 = env.step(st2, env.random_actions(st2))
        term = st2.terminated.cpu().numpy()
        rew = st2.rewards.cpu().numpy()
        mc = st2.game_state.move_count
        # PGX auto_reset: the terminating ply is reported (terminated, its
        # rewards) while the stored state is the reset env's
        assert (mc[term] == 0).all() and (mc[~term] == prev_mc[~term] + 1).all()
        assert not st2.game_state.terminated.any()
        assert (rew[~term] == 0).all()
        done += int(term.sum())
        assert not st2.truncated.cpu().numpy().any()
    assert done > 0
    assert (st2.game_state.move_count < 10).all()


def test_env_auto_reset_reports_draws_and_truncation():
    env = lx.LudaxEnvironment("pente", max_steps=6, auto_reset=True)
    st = env.init(seed=5, batch_size=40)
    for k in range(6):
        st = env.step_(st, env.RANDOM)
    assert st.terminated.all() and st.truncated.all() and not st.rewards.any()
    assert (st.game_state.move_count == 0).all()           # every row was reset


@pytest.mark.parametrize("name", ["tic_tac_toe", "connect_four", "reversi", "hex",
                                  "english_draughts", "yavalath"])
def test_env_random_step_equals_sample_then_step(name):
    a_env = lx.LudaxEnvironment(name, max_steps=200, auto_reset=True)
    b_env = lx.LudaxEnvironment(name, max_steps=200, auto_reset=True, mask_format="bits")
    B = 333
    sa = a_env.init(seed=8, batch_size=B)
    sb = b_env.init(seed=8, batch_size=B)
    for _ in range(60):
        acts = a_env.random_actions(sa)
        sa = a_env.step(sa, acts)
        sb = b_env.step(sb, b_env.RANDOM)
        assert torch.equal(sb.actions, acts)
        assert sa.game_state.digest() == sb.game_state.digest()
        assert torch.equal(sa.legal_action_mask, sb.mask_bool())
        for f in ("rewards", "terminated", "truncated", "current_player"):
            assert torch.equal(getattr(sa, f), getattr(sb, f)), f


def test_env_illegal_action_penalty_and_verify():
    env = lx.LudaxEnvironment("connect_four")
    st = env.init(seed=2, batch_size=8)
    acts = torch.full((8,), 38, dtype=torch.int64, device="cuda")   # bottom row: legal
    acts[5] = 3                                                      # top row: illegal
    acts[6] = 3
    d0 = st.game_state.digest()
    with pytest.raises(lx.errors.IllegalAction, match="row 5"):
        env.step(st, acts, verify=True)
    assert st.game_state.digest() == d0
    st2 = env.step(st, acts)
    assert st2.illegal_row() == 5
    t = st2.terminated.cpu().numpy()
    assert t.tolist() == [False] * 5 + [True, True, False]
    r = st2.rewards.cpu().numpy()
    assert r[5].tolist() == [-1.0, 1.0] and r[0].tolist() == [0.0, 0.0]   # P1 moved illegally
    assert st2.game_state.outcome[5] == 2
    ok = env.step(st, torch.full((8,), 38, dtype=torch.int64, device="cuda"))
    assert ok.illegal_row() is None


def test_env_truncation():
    env = lx.LudaxEnvironment("pente", max_steps=12)
    st = env.init(seed=3, batch_size=32)
    for _ in range(12):
        st = env.step(st, env.random_actions(st))
    assert st.truncated.all() and st.terminated.all() and not st.rewards.any()
