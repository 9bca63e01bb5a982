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
        st2 = env.step(st2, env.random_actions(st2))
        assert not st2.terminated.any()          # finished rows were reset
        done += int((st2.rewards != 0).any(dim=1).sum())
    assert done > 0
    assert (st2.game_state.move_count < 10).all()


def test_env_truncation():
    env = lx.LudaxEnvironment("pente", max_steps=12)
    st = env.init(seed=3, batch_size=32)
    for _ in range(12):
        st = env.step(st, env.random_actions(st))
    assert st.truncated.all() and st.terminated.all() and not st.rewards.any()
