"""PGX-style environment over a B200 game (BASELINE north star:
``LudaxEnvironment(game).init / step / legal_action_mask / rewards /
terminated``).

Everything stays on the device: ``EnvState`` fields are CUDA tensors and one
``step`` is one kernel launch (``lx_env_step``) that applies the actions (or,
with ``LudaxEnvironment.RANDOM``, samples a uniform legal action per env in
the same launch), rewards the terminating ply, truncates at ``max_steps``,
optionally auto-resets finished envs, and writes the next legal-action mask
-- as (B, A) bool, or bit-packed (B, ceil(A/32)) int32 with
``mask_format="bits"``.

Rewards follow the reference's outcome convention (engine.py:79-87,
agents.py:52-55): on the ply that ends the game, P1 win -> [+1, -1], P2 win
-> [-1, +1], draw -> [0, 0]; zero on every other ply.  With ``auto_reset``
the terminating ply's ``terminated`` / ``truncated`` / ``rewards`` are kept
while the state, mask and player are the reset env's (PGX auto_reset).  An
illegal action is never applied: ``step(..., verify=True)`` raises the
reference's IllegalAction (engine.step, mechanics.py:503-510) before any
change; unverified, the row ends with the PGX illegal-action penalty (mover
-1, opponent +1) and ``EnvState.illegal_row()`` names the lowest such row.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

from . import native
from .game import B200Game, DeviceState, _torch, load_config_game, load_game

ENV_AUTO_RESET, ENV_RANDOM, ENV_MASK_BITS, ENV_STEP = 1, 2, 4, 8     # include/ludax_b200.h


class _Random:
    def __repr__(self):
        return "LudaxEnvironment.RANDOM"


@dataclass
class EnvState:
    game_state: DeviceState           # bitboard SoA in HBM
    current_player: "object"          # (B,) int32
    legal_action_mask: "object"       # (B, A) bool, or None with mask_format="bits"
    rewards: "object"                 # (B, 2) float32
    terminated: "object"              # (B,) bool
    truncated: "object"               # (B,) bool
    legal_action_bits: "object" = None    # (B, ceil(A/32)) int32 with mask_format="bits"
    illegal: "object" = None          # (1,) int64 device: lowest illegal / stuck row, -1 none
    actions: "object" = None          # (B,) int64: the actions of the last RANDOM step

    @property
    def batch_size(self):
        return self.game_state.batch_size

    def illegal_row(self):
        """Lowest row whose last action was illegal (or, for a random step,
        that had no legal action and no pass); None when every row was fine.
        Synchronises."""
        if self.illegal is None:
            return None
        r = int(self.illegal.item())
        return None if r < 0 else r

    def mask_bool(self):
        """(B, A) bool legal mask in either format."""
        if self.legal_action_mask is not None:
            return self.legal_action_mask
        torch = _torch()
        A = self.game_state.game.action_space_size
        bits = self.legal_action_bits.view(torch.int32)
        shifts = torch.arange(32, device=bits.device, dtype=torch.int32)
        m = ((bits.unsqueeze(-1) >> shifts) & 1).bool()
        return m.reshape(bits.shape[0], -1)[:, :A]


class LudaxEnvironment:
    """``env = LudaxEnvironment(game_text | config name | B200Game)``."""

    RANDOM = _Random()                 # step_(state, env.RANDOM): sample in the step kernel

    def __init__(self, game, max_steps=0, auto_reset=False, mask_format="bool"):
        if isinstance(game, B200Game):
            self.game = game
        elif isinstance(game, str) and "(game" in game:
            self.game = load_game(game)
        elif isinstance(game, str):
            name = os.path.splitext(os.path.basename(game))[0]
            self.game = load_config_game(name)
        else:
            raise TypeError("game must be game text, a config game name or a B200Game")
        if mask_format not in ("bool", "bits"):
            raise ValueError("mask_format must be 'bool' or 'bits'")
        self.max_steps = int(max_steps)
        self.auto_reset = bool(auto_reset)
        self.mask_format = mask_format

    @property
    def num_actions(self):
        return self.game.action_space_size

    @property
    def mask_words(self):
        return (self.num_actions + 31) // 32

    @property
    def num_players(self):
        return 2

    @property
    def observation_shape(self):
        return (self.game.observation_planes, self.game.num_cells)

    def bytes_per_env_step(self, random=True):
        """Algorithmic HBM bytes of one env step: state read +
        write, mask, rewards, terminated, truncated, player (+ the action
        read when it is given)."""
        state = 2 * self.game.info["nq"] * 16
        mask = 4 * self.mask_words if self.mask_format == "bits" else self.num_actions
        return state + mask + 8 + 1 + 1 + 4 + (0 if random else 8)

    def _outputs(self, B):
        torch = _torch()
        if self.mask_format == "bits":
            mask = torch.empty((B, self.mask_words), dtype=torch.int32, device="cuda")
        else:
            mask = torch.empty((B, self.num_actions), dtype=torch.uint8, device="cuda")
        return (mask,
                torch.empty((B, 2), dtype=torch.float32, device="cuda"),
                torch.empty(B, dtype=torch.uint8, device="cuda"),
                torch.empty(B, dtype=torch.uint8, device="cuda"),
                torch.empty(B, dtype=torch.int32, device="cuda"),
                torch.empty(1, dtype=torch.int64, device="cuda"))

    def _state_outputs(self, state):
        torch = _torch()
        mask = (state.legal_action_bits if self.mask_format == "bits"
                else state.legal_action_mask.view(torch.uint8))
        illegal = state.illegal if state.illegal is not None else torch.empty(
            1, dtype=torch.int64, device="cuda")
        return (mask, state.rewards, state.terminated.view(torch.uint8),
                state.truncated.view(torch.uint8), state.current_player, illegal)

    def _launch(self, gs, flags, actions, out):
        torch = _torch()
        mask, rew, term, trunc, player, bad = out
        if self.auto_reset:
            flags |= ENV_AUTO_RESET
        if self.mask_format == "bits":
            flags |= ENV_MASK_BITS
        native.check(native.lib().lx_env_step(
            self.game.handle, gs.words.data_ptr(), gs.batch_size,
            actions.data_ptr() if actions is not None else None, self.max_steps, flags,
            mask.data_ptr(), rew.data_ptr(), term.data_ptr(), trunc.data_ptr(),
            player.data_ptr(), bad.data_ptr() if bad is not None else None,
            self.game._stream()))
        gs._touch()
        bits = self.mask_format == "bits"
        return EnvState(gs, player, None if bits else mask.view(torch.bool), rew,
                        term.view(torch.bool), trunc.view(torch.bool),
                        legal_action_bits=mask if bits else None, illegal=bad,
                        actions=actions if flags & ENV_RANDOM else None)

    def init(self, seed=0, batch_size=1, seeds=None):
        """Fresh batch; seeds spawn(seed, i) unless given (rng.py:52-54)."""
        gs = self.game.init(batch_size=batch_size, seed=seed, seeds=seeds)
        return self._launch(gs, 0, None, self._outputs(batch_size))

    def _actions(self, action, B):
        torch = _torch()
        a = action if isinstance(action, torch.Tensor) else torch.as_tensor(action)
        return a.to(device="cuda", dtype=torch.int64).reshape(-1).expand(B).contiguous()

    def _verify(self, gs, a):
        """Raise IllegalAction naming the first live row whose action is not
        legal (lx_step's verification pass, on a scratch copy of the state)."""
        import ctypes
        torch = _torch()
        scratch = torch.empty(1, dtype=torch.int64, device="cuda")
        bad = ctypes.c_int64(-1)
        st = native.lib().lx_step(self.game.handle, gs.words.data_ptr(), gs.batch_size,
                                  a.data_ptr(), None, 1, scratch.data_ptr(), ctypes.byref(bad),
                                  self.game._stream())
        native.check(st, bad.value)

    def step(self, state, action, verify=False):
        """Functional step: returns a new EnvState; ``state`` is not modified.
        ``action`` is a (B,) tensor / array / scalar or ``env.RANDOM``."""
        gs = state.game_state.copy()
        out = self._outputs(gs.batch_size)
        if action is self.RANDOM:
            acts = _torch().empty(gs.batch_size, dtype=_torch().int64, device="cuda")
            return self._launch(gs, ENV_STEP | ENV_RANDOM, acts, out)
        a = self._actions(action, gs.batch_size)
        if verify:
            self._verify(gs.copy(), a)
        return self._launch(gs, ENV_STEP, a, out)

    def step_(self, state, action, out=None, verify=False):
        """In-place step reusing ``state``'s output buffers (no allocation for
        ``env.RANDOM``): one kernel launch per ply."""
        out = out if out is not None else self._state_outputs(state)
        if action is self.RANDOM:       # hot path: no illegal-row flag (no memset per ply)
            return self._launch(state.game_state, ENV_STEP | ENV_RANDOM, None,
                                out[:5] + (None,))
        a = self._actions(action, state.batch_size)
        if verify:
            self._verify(state.game_state.copy(), a)
        return self._launch(state.game_state, ENV_STEP, a, out)

    def observe(self, state, player=None):
        """(B, 2T+1, C) bool planes for ``player`` (default: each row's mover is
        not batched -- pass a player id) (compiler.py:611-626)."""
        p = 0 if player is None else int(player)
        return self.game.observe_device(state.game_state, p)

    def random_actions(self, state):
        """Uniform legal actions from each env's own counter stream (the
        actions ``step_(state, env.RANDOM)`` samples in its kernel)."""
        return self.game.sample_actions_device(state.game_state)


__all__ = ["LudaxEnvironment", "EnvState"]
