"""PGX-style environment over a B200 game (BASELINE north star:
``LudaxEnvironment(game).init / step / legal_action_mask / rewards /
terminated``).

Everything stays on the device: ``EnvState`` fields are CUDA tensors and one
``step`` is one kernel launch (``lx_env_step``) that applies the actions,
rewards the terminating ply, truncates at ``max_steps``, optionally
auto-resets finished envs, and writes the next legal-action mask.

Rewards follow the reference's outcome convention (engine.py:79-87,
agents.py:52-55): on the ply that ends the game, P1 win -> [+1, -1], P2 win
-> [-1, +1], draw -> [0, 0]; zero on every other ply.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

from . import native
from .game import B200Game, DeviceState, _torch, load_config_game, load_game


@dataclass
class EnvState:
    game_state: DeviceState           # bitboard SoA in HBM
    current_player: "object"          # (B,) int32
    legal_action_mask: "object"       # (B, A) bool
    rewards: "object"                 # (B, 2) float32
    terminated: "object"              # (B,) bool
    truncated: "object"               # (B,) bool

    @property
    def batch_size(self):
        return self.game_state.batch_size


class LudaxEnvironment:
    """``env = LudaxEnvironment(game_text | config name | B200Game)``."""

    def __init__(self, game, max_steps=0, auto_reset=False):
        if isinstance(game, B200Game):
            self.game = game
        elif isinstance(game, str) and "(game" in game:
            self.game = load_game(game)
        elif isinstance(game, str):
            name = os.path.splitext(os.path.basename(game))[0]
            self.game = load_config_game(name)
        else:
            raise TypeError("game must be game text, a config game name or a B200Game")
        self.max_steps = int(max_steps)
        self.auto_reset = bool(auto_reset)

    @property
    def num_actions(self):
        return self.game.action_space_size

    @property
    def num_players(self):
        return 2

    @property
    def observation_shape(self):
        return (self.game.observation_planes, self.game.num_cells)

    def _outputs(self, B):
        torch = _torch()
        return (torch.empty((B, self.num_actions), dtype=torch.uint8, device="cuda"),
                torch.empty((B, 2), dtype=torch.float32, device="cuda"),
                torch.empty(B, dtype=torch.uint8, device="cuda"),
                torch.empty(B, dtype=torch.uint8, device="cuda"),
                torch.empty(B, dtype=torch.int32, device="cuda"))

    def _launch(self, gs, actions, out):
        torch = _torch()
        mask, rew, term, trunc, player = out
        native.check(native.lib().lx_env_step(
            self.game.handle, gs.words.data_ptr(), gs.batch_size,
            actions.data_ptr() if actions is not None else None, self.max_steps,
            int(self.auto_reset), mask.data_ptr(), rew.data_ptr(), term.data_ptr(),
            trunc.data_ptr(), player.data_ptr(), self.game._stream()))
        gs._touch()
        return EnvState(gs, player, mask.view(torch.bool), rew, term.view(torch.bool),
                        trunc.view(torch.bool))

    def init(self, seed=0, batch_size=1, seeds=None):
        """Fresh batch; seeds spawn(seed, i) unless given (rng.py:52-54)."""
        gs = self.game.init(batch_size=batch_size, seed=seed, seeds=seeds)
        return self._launch(gs, None, self._outputs(batch_size))

    def step(self, state, action):
        """Functional step: returns a new EnvState; ``state`` is not modified."""
        torch = _torch()
        gs = state.game_state.copy()
        a = action if isinstance(action, torch.Tensor) else torch.as_tensor(action)
        a = a.to(device="cuda", dtype=torch.int64).reshape(-1).expand(gs.batch_size).contiguous()
        return self._launch(gs, a, self._outputs(gs.batch_size))

    def step_(self, state, action, out=None):
        """In-place step (no state copy, optional reused output buffers)."""
        torch = _torch()
        a = action if isinstance(action, torch.Tensor) else torch.as_tensor(action)
        a = a.to(device="cuda", dtype=torch.int64).contiguous()
        if out is None:
            out = (state.legal_action_mask.view(torch.uint8), state.rewards,
                   state.terminated.view(torch.uint8), state.truncated.view(torch.uint8),
                   state.current_player)
        return self._launch(state.game_state, a, out)

    def observe(self, state, player=None):
        """(B, 2T+1, C) bool planes for ``player`` (default: each row's mover is
        not batched -- pass a player id) (compiler.py:611-626)."""
        p = 0 if player is None else int(player)
        return self.game.observe_device(state.game_state, p)

    def random_actions(self, state):
        """Uniform legal actions from each env's own counter stream."""
        return self.game.sample_actions_device(state.game_state)


__all__ = ["LudaxEnvironment", "EnvState"]
