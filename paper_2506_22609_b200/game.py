"""B200Game: the CompiledGame-compatible face of one lowered game, and
DeviceState: a batch of envs held as bitboard SoA in HBM.

Drop-in surface (reference: pkg/src/boardlang/compiler.py:197-650):
``init``, ``legal_mask``, ``legal_counts``, ``sample_actions``, ``step``,
``step_into``, ``observe``, ``describe``, ``codec``, ``layout``,
``action_space_size``, ``pass_index``.  Host-facing methods accept and
return numpy arrays exactly like the reference; every computation runs in
the game's sm_100a kernels.  ``*_device`` variants keep inputs and outputs
as CUDA tensors for zero-copy pipelines (``env.LudaxEnvironment``).

A DeviceState answers the reference GameState attribute names
(``board_owner``, ``terminated``, ``scores``, ... state.py:78-130) by
exporting the device words through ``lx_export`` on first access, so
reference-style code (``state.terminated.all()``, ``state.digest()``)
works unchanged.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from dataclasses import dataclass

import numpy as np

from . import errors, native
from .errors import CompileError, EmptyMask
from .lowering import lower_game
from .syntax import parse_game

GAMES_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "games")
MCTS_SHARED_LIMIT = 200 * 1024      # dynamic shared memory per MCTS tree (B200 opt-in 227 KB; the runtime checks it with the kernel's static buffers)

# per-cell planes: exported read-only (DeviceState.host)
READONLY_FIELDS = ("board_piece", "board_owner", "comp_labels", "hopped_mask", "captured_mask",
                   "promoted_mask")

FIELDS = ("board_piece", "board_owner", "current_player", "move_count", "terminated",
          "truncated", "outcome", "seeds", "scores", "pass_streak", "pass_flags", "must_move",
          "last_mover", "last_kind", "last_source", "last_dest", "last_dest_by_player",
          "hopped_mask", "captured_mask", "promoted_mask", "comp_labels", "phase", "turn_pos")


_TORCH = None


def _torch():
    # checked once per process (torch.cuda.is_available reads the environment
    # on every call: ~4 us, hundreds of calls per MCTS match)
    global _TORCH
    if _TORCH is None:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2506_22609_b200 needs a CUDA device (sm_100a); "
                               "there is no CPU fallback")
        _TORCH = torch
    return _TORCH


@dataclass(frozen=True)
class ActionCodec:
    """Action index <-> move (reference codec.py:16-69): placement = cell,
    movement = source * C + dest, gridworld = direction index; optional
    trailing pass."""
    kind: str
    num_cells: int
    size: int
    has_pass: bool
    directions: tuple = ()

    @property
    def pass_index(self):
        return self.size - 1 if self.has_pass else None

    def encode(self, source, dest):
        if self.kind == "movement":
            return source * self.num_cells + dest
        if self.kind == "placement":
            return dest
        raise ValueError("gridworld actions are direction indices; use encode_direction")

    def encode_direction(self, direction):
        return self.directions.index(direction)

    def decode(self, action):
        if self.has_pass and action == self.pass_index:
            return None, None
        if self.kind == "movement":
            return action // self.num_cells, action % self.num_cells
        if self.kind == "placement":
            return None, action
        return None, None

    def describe(self, action):
        if self.has_pass and action == self.pass_index:
            return {"kind": "pass"}
        if self.kind == "movement":
            return {"kind": "move", "source": action // self.num_cells,
                    "dest": action % self.num_cells}
        if self.kind == "placement":
            return {"kind": "place", "dest": action}
        return {"kind": "direction", "direction": self.directions[action]}


@dataclass(frozen=True)
class StateLayout:
    """Which reference GameState fields this game materialises (state.py:34-66)."""
    scores: bool = False
    passing: bool = False
    must_move: bool = False
    last_action: bool = False
    transient_masks: bool = False
    connectivity: int = 0
    phase: bool = False
    turn_pos: bool = False


class DeviceState:
    """Batch of envs in HBM: int32 words shaped (NQ, B, 4), quad-major.

    Reading a reference GameState field (``state.terminated``,
    ``state.board_owner``, ... state.py:78-130) exports the device words once
    (lx_export) into a host cache; in-place edits of those arrays -- what the
    reference's own loops do, e.g. ``state.terminated |= truncate`` and
    ``state.outcome[rows] = 0`` (engine.py:156-160) -- are written back to the
    device (lx_import) before the next device call that reads the state, so
    reference-style code sees value semantics.  Device calls that change the
    state drop the cache.
    """

    def __init__(self, game, words, batch_size):
        self.game = game
        self.words = words
        self.batch_size = batch_size
        self._host = None
        self._snap = None

    # -- value semantics --
    def copy(self):
        self.sync()
        return DeviceState(self.game, self.words.clone(), self.batch_size)

    def _touch(self):
        self._host = None
        self._snap = None

    def sync(self):
        """Write host-side edits of the cached reference fields back to the
        device (no-op when nothing was read or nothing changed)."""
        if self._host is None:
            return
        if all(np.array_equal(self._host[k], v) for k, v in self._snap.items()):
            return
        self.game._import_into(self, self._host)
        self._snap = {k: self._host[k].copy() for k in self._snap}

    # -- reference field view --
    def host(self):
        """dict of numpy arrays in the reference GameState layout.  The
        per-env scalar fields are writable (edits reach the device, see the
        class docstring); the per-cell planes (boards, component labels,
        transient masks) are read-only views, so an in-place edit of them
        raises instead of being lost -- and the change check copies only the
        scalar fields (~25 B/env, not the ~110-760 B/env of the planes)."""
        if self._host is None:
            self._host = self.game._export(self)
            for k in READONLY_FIELDS:
                if self._host.get(k) is not None:
                    self._host[k].setflags(write=False)
            self._snap = {k: v.copy() for k, v in self._host.items()
                          if k not in READONLY_FIELDS}
        return self._host

    def __getattr__(self, name):
        if name in FIELDS:
            return self.host().get(name)
        raise AttributeError(name)

    def digest(self):
        """Same bytes as the reference GameState.digest (state.py:180-188)."""
        h = hashlib.blake2b(digest_size=16)
        host = self.host()
        for name in FIELDS:
            v = host.get(name)
            if v is not None:
                h.update(name.encode())
                h.update(np.ascontiguousarray(v).tobytes())
        return h.hexdigest()

    def nbytes(self):
        return sum(v.nbytes for v in self.host().values())

    def device_nbytes(self):
        return self.words.numel() * 4

    def rows(self, idx):
        self.sync()
        idx = np.atleast_1d(np.asarray(idx))
        torch = _torch()
        t = torch.as_tensor(idx, device=self.words.device, dtype=torch.long)
        return DeviceState(self.game, self.words[:, t].contiguous(), len(idx))

    @classmethod
    def concat(cls, states):
        torch = _torch()
        for s in states:
            s.sync()
        w = torch.cat([s.words for s in states], dim=1).contiguous()
        return cls(states[0].game, w, sum(s.batch_size for s in states))

    def set_rows(self, idx, other):
        torch = _torch()
        self.sync()
        other.sync()
        t = torch.as_tensor(np.atleast_1d(np.asarray(idx)), device=self.words.device,
                            dtype=torch.long)
        self.words[:, t] = other.words
        self._touch()

    def equal(self, other):
        return self.digest() == other.digest()


class B200Game:
    """One game lowered to sm_100a kernels (CompiledGame drop-in)."""

    def __init__(self, spec, text=None):
        self.spec = spec
        lowered = lower_game(spec)
        self.lowered = lowered
        self.info = lowered.info
        self.name = spec.name
        self.num_cells = lowered.info["C"]
        L = lowered.info["layout"]
        self.layout = StateLayout(**{k: L[k] for k in StateLayout.__dataclass_fields__})
        self.codec = ActionCodec(lowered.info["codec"], self.num_cells, lowered.info["A"],
                                 lowered.info["pass_index"] >= 0,
                                 tuple(lowered.info["grid_directions"]))
        self.piece_names = tuple(p.name for p in spec.equipment.pieces)
        self._native = {}
        self._nq = lowered.info["nq"]

    # -- native handle (lazy: needs the CUDA context) --
    @property
    def native(self):
        """The lx_game handle of the current device (one per device: a handle
        is bound to the device whose context was current at creation)."""
        dev = _torch().cuda.current_device()
        h = self._native.get(dev)
        if h is None:
            # torch's current device may not have made its (primary) context
            # current on this thread yet; the handle binds to that context
            native.check(native.lib().lx_bind_device(dev))
            i = self.lowered.info
            h = native.NativeGame(self.lowered.source, self.name, expect={
                "num_cells": i["C"], "num_actions": i["A"], "pass_index": i["pass_index"],
                "board_words": i["W"], "state_quads": i["nq"], "private_words": i["NX"],
                "mechanics": i["mechanics"], "device": dev})
            self._native[dev] = h
        return h

    @property
    def handle(self):
        return self.native.h

    def lowered_key(self):
        """NVRTC cache key: generated unit + device headers + options (profiles
        under profiles/ are keyed on it)."""
        return native.cache_key(self.lowered.source)

    @staticmethod
    def _stream():
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    @property
    def action_space_size(self):
        return self.codec.size

    @property
    def pass_index(self):
        return self.codec.pass_index

    @property
    def observation_planes(self):
        return 2 * len(self.piece_names) + 1

    def describe(self):
        b = self.spec.equipment.board
        return {"name": self.name,
                "board": {"kind": b.kind, "rows": b.rows, "cols": b.cols},
                "num_cells": self.num_cells, "pieces": list(self.piece_names),
                "action_space": {"kind": self.codec.kind, "size": self.codec.size,
                                 "has_pass": self.codec.has_pass},
                "observation_planes": self.observation_planes,
                "phases": len(self.spec.phases),
                "state_layout": {"scores": self.layout.scores, "passing": self.layout.passing,
                                 "must_move": self.layout.must_move,
                                 "last_action": self.layout.last_action,
                                 "transient_masks": self.layout.transient_masks,
                                 "connectivity_plans": self.layout.connectivity,
                                 "phase_index": self.layout.phase,
                                 "turn_position": self.layout.turn_pos},
                "state_bytes": self.reference_state_bytes(),
                "device_state_bytes": self._nq * 16}

    def reference_state_bytes(self):
        """Bytes per env of the reference GameState layout (the reference's
        describe()["state_bytes"], compiler.py:649): the fields this game's
        StateLayout materialises (state.py:34-130)."""
        C, L = self.num_cells, self.layout
        n = 2 * C + 1 + 4 + 1 + 1 + 1 + 8          # boards, player, mc, term, trunc, outcome, seed
        n += 8 if L.scores else 0
        n += 2 + 2 if L.passing else 0
        n += 2 if L.must_move else 0
        n += 1 + 1 + 2 + 2 + 4 if L.last_action else 0
        n += 3 * C if L.transient_masks else 0
        n += 2 * C * L.connectivity
        n += 1 if L.phase else 0
        n += 1 if L.turn_pos else 0
        return n

    # -- allocation --
    def empty_state(self, B):
        torch = _torch()
        w = torch.empty((self._nq, B, 4), dtype=torch.int32, device="cuda")
        return DeviceState(self, w, B)

    def init(self, batch_size=1, seed=0, seeds=None, first_index=0):
        """CompiledGame.init (compiler.py:357-364); seeds spawned on device."""
        torch = _torch()
        st = self.empty_state(batch_size)
        seeds_t = None
        if seeds is not None:
            seeds_t = _u64_tensor(seeds, batch_size)
        native.check(native.lib().lx_init(
            self.handle, st.words.data_ptr(), batch_size,
            seeds_t.data_ptr() if seeds_t is not None else None,
            int(seed) & (2 ** 64 - 1), int(first_index), self._stream()))
        del torch
        return st

    def occupied_device(self, state):
        """(B, C) bool CUDA tensor: cells holding a stone (board_owner >= 0),
        exported on the device without a host copy (play_match coverage)."""
        torch = _torch()
        state.sync()
        B, C = state.batch_size, self.num_cells
        buf = torch.empty((2, B, C), dtype=torch.int8, device="cuda")
        ref = native.RefState(board_owner=buf[0].data_ptr(), board_piece=buf[1].data_ptr())
        native.check(native.lib().lx_export(self.handle, state.words.data_ptr(), B,
                                            ctypes.byref(ref), self._stream()))
        return buf[0] >= 0

    # -- per-row scalars (lx_export of the scalar fields only) --
    def meta(self, state, counts=False):
        """Host numpy arrays of current_player, move_count, terminated,
        truncated, outcome and seeds (one export launch, no boards) -- and,
        with ``counts``, the legal action counts (one lx_legal launch) -- in
        one device-to-host copy."""
        state.sync()
        torch = _torch()
        B = state.batch_size
        nb = 24 * B if counts else 16 * B
        buf = torch.empty(nb, dtype=torch.uint8, device="cuda")
        o = buf.data_ptr()
        # [seeds u64 | counts i64 | move_count i32 | player | terminated | truncated | outcome]
        c = 8 * B if counts else 0
        ref = native.RefState(seeds=o, move_count=o + c + 8 * B, current_player=o + c + 12 * B,
                              terminated=o + c + 13 * B, truncated=o + c + 14 * B,
                              outcome=o + c + 15 * B)
        native.check(native.lib().lx_export(self.handle, state.words.data_ptr(), B,
                                            ctypes.byref(ref), self._stream()))
        if counts:
            native.check(native.lib().lx_legal(self.handle, state.words.data_ptr(), B, None,
                                               None, o + 8 * B, self._stream()))
        h = buf.cpu().numpy()
        out = {"seeds": h[:8 * B].view(np.uint64).copy(),
               "move_count": h[c + 8 * B:c + 12 * B].view(np.int32).copy(),
               "current_player": h[c + 12 * B:c + 13 * B].view(np.int8).copy(),
               "terminated": h[c + 13 * B:c + 14 * B].astype(bool),
               "truncated": h[c + 14 * B:c + 15 * B].astype(bool),
               "outcome": h[c + 15 * B:c + 16 * B].view(np.int8).copy()}
        if counts:
            out["legal_counts"] = h[8 * B:16 * B].view(np.int64).copy()
        return out

    def expand(self, pool_words, cap, parents, actions, children, seeds, max_turns,
               masks=True):
        """MCTS expansion + rollouts in one launch (lx_expand): children rows of
        the node pool get their parents' states stepped with `actions`; returns
        host arrays (info int32, rolled int8, masks (n, A) bool or None) --
        one host->device and one device->host copy."""
        torch = _torch()
        n = len(parents)
        A = self.codec.size
        nb = 4 * n + n + (n * A if masks else 0)
        bufs = getattr(self, "_xbufs", None)        # pinned + device staging, reused
        if bufs is None or bufs[0].numel() < 4 * n or bufs[2].numel() < nb:
            cap_in, cap_out = max(4 * n, 4096), max(nb, 1 << 16)
            bufs = (torch.empty(cap_in, dtype=torch.int64).pin_memory(),
                    torch.empty(cap_in, dtype=torch.int64, device="cuda"),
                    torch.empty(cap_out, dtype=torch.uint8).pin_memory(),
                    torch.empty(cap_out, dtype=torch.uint8, device="cuda"))
            self._xbufs = bufs
        pin_in, dev_in, pin_out, dev_out = bufs
        host = pin_in.numpy()
        host[:n] = parents
        host[n:2 * n] = actions
        host[2 * n:3 * n] = children
        host[3 * n:4 * n] = np.asarray(seeds, dtype=np.uint64).view(np.int64)
        dev_in[:4 * n].copy_(pin_in[:4 * n], non_blocking=True)
        p = dev_in.data_ptr()
        o = dev_out.data_ptr()
        native.check(native.lib().lx_expand(
            self.handle, pool_words.data_ptr(), int(cap), p, p + 8 * n, p + 16 * n, n, p + 24 * n,
            int(max_turns), o, o + 4 * n, (o + 5 * n) if masks else None, self._stream()))
        pin_out[:nb].copy_(dev_out[:nb], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        h = pin_out.numpy()
        return (h[:4 * n].view(np.int32).copy(), h[4 * n:5 * n].view(np.int8).copy(),
                h[5 * n:nb].reshape(n, A).astype(bool) if masks else None)

    def mcts(self, roots, keys, budgets, exploration, rollout_max_turns):
        """One MCTS decision per root row on the device (lx_mcts, one warp
        per tree, the tree in shared memory when it fits).  Returns (actions int64, ok bool) host arrays; rows with
        ok False exceeded a capacity and must be searched on the host."""
        roots.sync()
        import math
        torch = _torch()
        n = roots.batch_size
        budgets = np.asarray(budgets, dtype=np.int32)
        nmax = int(budgets.max()) + 2
        A = self.codec.size
        node_bytes = 40                                   # lx::MctsNode
        arena_bytes = nmax * node_bytes + 8 * (A + 1 + nmax * min(A, 256)) + 12 * (A + 1)
        arena_bytes = (arena_bytes + 15) // 16 * 16
        # the whole tree in shared memory when it fits the opt-in limit
        shared = arena_bytes + nmax * self._nq * 16
        shared = shared if shared <= MCTS_SHARED_LIMIT else 0
        cache = getattr(self, "_mcts_logs", None)
        if cache is None or cache.numel() < nmax + 2:
            cache = torch.tensor([0.0] + [math.log(k) for k in range(1, nmax + 2)],
                                 dtype=torch.float64, device="cuda")
            self._mcts_logs = cache
        logs = cache
        keys_t = _u64_tensor(keys, n)
        bud_t = torch.as_tensor(budgets).to("cuda")
        if shared:
            pool = torch.empty(1, dtype=torch.int32, device="cuda")
            arena = torch.empty(1, dtype=torch.uint8, device="cuda")
        else:
            pool = torch.empty((self._nq, n * nmax, 4), dtype=torch.int32, device="cuda")
            arena = torch.empty(n * arena_bytes, dtype=torch.uint8, device="cuda")
        out = torch.empty(3 * n, dtype=torch.int32, device="cuda")   # actions (i64) | status
        acts, status = out[:2 * n].view(torch.int64), out[2 * n:]
        st = native.lib().lx_mcts(
            self.handle, roots.words.data_ptr(), n, keys_t.data_ptr(), bud_t.data_ptr(),
            float(exploration), int(rollout_max_turns), logs.data_ptr(), int(logs.numel()),
            pool.data_ptr(), n * nmax, nmax, arena.data_ptr(), arena_bytes, acts.data_ptr(),
            status.data_ptr(), int(shared), self._stream())
        if st == errors.LX_EINVALID and shared:   # the tree does not fit next to the
            pool = torch.empty((self._nq, n * nmax, 4), dtype=torch.int32, device="cuda")
            arena = torch.empty(n * arena_bytes, dtype=torch.uint8, device="cuda")
            st = native.lib().lx_mcts(     # kernel's static shared buffers: global arena
                self.handle, roots.words.data_ptr(), n, keys_t.data_ptr(), bud_t.data_ptr(),
                float(exploration), int(rollout_max_turns), logs.data_ptr(), int(logs.numel()),
                pool.data_ptr(), n * nmax, nmax, arena.data_ptr(), arena_bytes, acts.data_ptr(),
                status.data_ptr(), 0, self._stream())
        native.check(st)
        h = out.cpu().numpy()
        return h[:2 * n].view(np.int64).copy(), h[2 * n:] == 0

    def truncate_rows(self, state, rows):
        """Mark rows terminated + truncated with a draw outcome in place (the
        reference's stuck / turn-cap handling, engine.py:156-160,
        agents.py:430-435)."""
        state.sync()
        torch = _torch()
        r = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.uint8)).to("cuda")
        native.check(native.lib().lx_truncate(self.handle, state.words.data_ptr(),
                                              state.batch_size, r.data_ptr(), self._stream()))
        state._touch()

    def _device(self, state):
        """DeviceState for a state argument: itself (host edits written back),
        or a reference GameState-like object imported with lx_import."""
        arrays = _foreign_arrays(state)
        if arrays is None:
            return _sync(state)
        return self.from_reference(arrays)

    # -- legality / sampling --
    def _mover_tensor(self, mover, state):
        if mover is None:
            return None
        torch = _torch()
        m = mover if isinstance(mover, torch.Tensor) else torch.as_tensor(
            np.broadcast_to(np.asarray(mover), (state.batch_size,)).astype(np.int8))
        return m.to(device="cuda", dtype=torch.int8).reshape(-1).expand(
            state.batch_size).contiguous()

    def legal_mask_device(self, state, mover=None):
        torch = _torch()
        B = state.batch_size
        mv = self._mover_tensor(mover, state)
        mask = torch.empty((B, self.codec.size), dtype=torch.uint8, device="cuda")
        native.check(native.lib().lx_legal(self.handle, state.words.data_ptr(), B,
                                           mv.data_ptr() if mv is not None else None,
                                           mask.data_ptr(), None, self._stream()))
        return mask.view(torch.bool)

    def legal_counts_device(self, state, mover=None):
        torch = _torch()
        B = state.batch_size
        mv = self._mover_tensor(mover, state)
        counts = torch.empty(B, dtype=torch.int64, device="cuda")
        native.check(native.lib().lx_legal(self.handle, state.words.data_ptr(), B,
                                           mv.data_ptr() if mv is not None else None, None,
                                           counts.data_ptr(), self._stream()))
        return counts

    def legal_mask(self, state, mover=None):
        """(B, A) bool numpy; all-false for terminated rows (compiler.py:411-428).
        ``mover``: (B,) player ids (or a scalar) whose legal actions to list
        instead of each row's current player."""
        state = self._device(state)
        return self.legal_mask_device(state, mover).cpu().numpy()

    def legal_counts(self, state, mover=None):
        """(B,) int64 legal action counts, pass included (compiler.py:394-409)."""
        state = self._device(state)
        return self.legal_counts_device(state, mover).cpu().numpy()

    def sample_actions_device(self, state, u=None, mover=None):
        torch = _torch()
        B = state.batch_size
        mv = self._mover_tensor(mover, state)
        out = torch.empty(B, dtype=torch.int64, device="cuda")
        u_t = None
        if u is not None:
            u_t = u if isinstance(u, torch.Tensor) else torch.as_tensor(
                np.ascontiguousarray(u, dtype=np.float64))
            u_t = u_t.to(device="cuda", dtype=torch.float64).contiguous()
        native.check(native.lib().lx_sample(self.handle, state.words.data_ptr(), B,
                                            mv.data_ptr() if mv is not None else None,
                                            u_t.data_ptr() if u_t is not None else None,
                                            out.data_ptr(), self._stream()))
        return out

    def sample_actions(self, state, u, mover=None):
        """Uniform legal action per row from a (B,) float64 draw (compiler.py:430-446)."""
        state = self._device(state)
        return self.sample_actions_device(state, u, mover).cpu().numpy()

    # -- stepping --
    def step(self, state, actions):
        """Pure step (compiler.py:450-454): copy, then verified step_into."""
        out = self._device(state)
        out = out.copy() if out is state else out
        self.step_into(out, actions, verify=True)
        return out

    def step_into(self, state, actions, rows=None, verify=True):
        """In-place step on rows & ~terminated (compiler.py:456-580).  A
        reference GameState-like argument is imported, stepped on the device
        and its arrays overwritten in place with the result."""
        foreign = _foreign_arrays(state)
        if foreign is not None:
            dev = self.from_reference(foreign)
            self.step_into(dev, actions, rows=rows, verify=verify)
            for k, v in dev.host().items():
                cur = getattr(state, k, None)
                if cur is not None:
                    cur[...] = v
            if hasattr(state, "_mech_cache"):
                state._mech_cache = None
            return
        state.sync()
        torch = _torch()
        B = state.batch_size
        a = actions if isinstance(actions, torch.Tensor) else torch.as_tensor(
            np.broadcast_to(np.asarray(actions, dtype=np.int64), (B,)).copy())
        a = a.to(device="cuda", dtype=torch.int64).contiguous()
        r = None
        if rows is not None:
            r = rows if isinstance(rows, torch.Tensor) else torch.as_tensor(
                np.ascontiguousarray(rows, dtype=bool))
            r = r.to(device="cuda", dtype=torch.uint8).contiguous()
        scratch = torch.empty(1, dtype=torch.int64, device="cuda") if verify else None
        bad = ctypes.c_int64(-1)
        st = native.lib().lx_step(self.handle, state.words.data_ptr(), B, a.data_ptr(),
                                  r.data_ptr() if r is not None else None, int(bool(verify)),
                                  scratch.data_ptr() if scratch is not None else None,
                                  ctypes.byref(bad), self._stream())
        native.check(st, bad.value)
        state._touch()

    def random_step(self, state, max_turns=200, record=False):
        """One fused uniform-random ply for live rows; returns actions if record."""
        state.sync()
        torch = _torch()
        B = state.batch_size
        out = torch.empty(B, dtype=torch.int64, device="cuda") if record else None
        native.check(native.lib().lx_random_step(self.handle, state.words.data_ptr(), B,
                                                 int(max_turns),
                                                 out.data_ptr() if out is not None else None,
                                                 self._stream()))
        state._touch()
        return out

    def rollout(self, batch_size=None, seed=0, seeds=None, state=None, max_turns=200,
                store=True, truncate=True, first_index=0, check=True, stats=None, work=None,
                outcomes=None, turns=None, out=None):
        """Fused register-resident rollout (kernel lx_rollout).

        Without ``state``: envs start from ``seeds`` (or spawn(seed, first_index+i))
        and, with ``store``, the final states are written to ``out`` (allocated
        when None) and returned.  With ``state``: continue those envs in place.
        Returns (final DeviceState or None, stats tensor u64[8]: steps, p1, p2,
        draws, truncated, envs).
        """
        torch = _torch()
        mode = 0
        if state is None:
            mode |= 1
            B = int(batch_size) if batch_size is not None else (
                out.batch_size if out is not None else len(seeds))
            if store:
                state = out if out is not None else self.empty_state(B)
        else:
            state.sync()
            B = state.batch_size
        if store:
            mode |= 2
        if truncate:
            mode |= 4
        seeds_t = _u64_tensor(seeds, B) if seeds is not None else None
        if stats is None:
            stats = torch.empty(8, dtype=torch.int64, device="cuda")
        if work is None:
            work = torch.zeros(16, dtype=torch.int64, device="cuda")    # LX_ROLLOUT_WORK_BYTES
        stuck = ctypes.c_int64(-1)
        st = native.lib().lx_rollout(
            self.handle, state.words.data_ptr() if state is not None else None, B,
            int(max_turns), mode, int(seed) & (2 ** 64 - 1),
            seeds_t.data_ptr() if seeds_t is not None else None, int(first_index),
            stats.data_ptr(), work.data_ptr(),
            outcomes.data_ptr() if outcomes is not None else None,
            turns.data_ptr() if turns is not None else None,
            int(bool(check)), ctypes.byref(stuck),
            self._stream())
        native.check(st, stuck.value)
        if state is not None:
            state._touch()
        return state, stats

    def _host_playout_args(self, batch_size, seed, seeds, first_index, outcomes, turns, stats,
                           out):
        torch = _torch()

        def host_ptr(a, dtype, n, what):
            if a is None or a is False:
                return None, None
            if a is True:
                a = np.empty(n, dtype=dtype)
            if isinstance(a, torch.Tensor):
                if a.is_cuda or not a.is_contiguous() or a.numel() != n or \
                        a.element_size() != np.dtype(dtype).itemsize:
                    raise ValueError(f"{what}: need a contiguous host tensor of {n} "
                                     f"{np.dtype(dtype).name}")
                return a, a.data_ptr()
            a = np.asarray(a)
            if not (a.flags.c_contiguous and a.size == n and a.dtype.itemsize ==
                    np.dtype(dtype).itemsize):
                raise ValueError(f"{what}: need a contiguous host array of {n} "
                                 f"{np.dtype(dtype).name}")
            return a, a.ctypes.data
        if batch_size is not None:
            B = int(batch_size)
        elif seeds is not None:
            B = len(seeds)
        elif out is not None:
            B = out.batch_size
        else:
            raise ValueError("batch_size, seeds or out is required")
        if seeds is not None and not isinstance(seeds, torch.Tensor):
            seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        return B, (host_ptr(seeds, np.uint64, B, "seeds"),
                   host_ptr(outcomes, np.int8, B, "outcomes"),
                   host_ptr(turns, np.int32, B, "turns"),
                   host_ptr(stats if stats is not None else True, np.uint64, 8, "stats"))

    def playout_host(self, batch_size=None, seed=0, seeds=None, first_index=0, max_turns=200,
                     truncate=True, outcomes=True, turns=False, stats=None, out=None,
                     upload_first=False):
        """One batch episode through the host-buffer C-ABI call lx_playout_host
        (the reference's evaluation._run_episode / engine.playout_random as a
        numpy caller binds them, evaluation.py:197-211, engine.py:123-163):
        per-env seeds in host memory (numpy or a pinned torch CPU tensor; None:
        spawn(seed, first_index + i)), outcomes / final move counts / stats
        back in host memory.  ``outcomes`` / ``turns``: True to allocate,
        a host array to fill, or False; ``out``: optional DeviceState for the
        final states.  The seed upload overlaps the play (see the header).
        Returns (outcomes or None, turns or None, stats (8,) uint64)."""
        B, (sd, oc, tn, st_) = self._host_playout_args(batch_size, seed, seeds, first_index,
                                                       outcomes, turns, stats, out)
        flags = (1 if truncate else 0) | (2 if upload_first else 0)
        stuck = ctypes.c_int64(-1)
        st = native.lib().lx_playout_host(
            self.handle, B, int(max_turns), flags, int(seed) & (2 ** 64 - 1), sd[1],
            int(first_index), oc[1], tn[1], st_[1],
            out.words.data_ptr() if out is not None else None, ctypes.byref(stuck),
            self._stream())
        if out is not None:
            out._touch()
        native.check(st, stuck.value)
        return oc[0], tn[0], st_[0]

    def playout_host_async(self, batch_size=None, seed=0, seeds=None, first_index=0,
                           max_turns=200, truncate=True, outcomes=True, turns=False, stats=None,
                           out=None):
        """lx_playout_host_async: enqueue one host-buffer episode and return a
        ticket for playout_host_wait (two episodes in flight per handle: the
        next one's seed upload and the previous one's download overlap this
        one's rollout).  Host buffers should be pinned torch tensors."""
        B, (sd, oc, tn, st_) = self._host_playout_args(batch_size, seed, seeds, first_index,
                                                       outcomes, turns, stats, out)
        ticket = ctypes.c_int64(-1)
        native.check(native.lib().lx_playout_host_async(
            self.handle, B, int(max_turns), 1 if truncate else 0, int(seed) & (2 ** 64 - 1),
            sd[1], int(first_index), oc[1], tn[1], st_[1],
            out.words.data_ptr() if out is not None else None, self._stream(),
            ctypes.byref(ticket)))
        if out is not None:
            out._touch()
        # the arrays ride along so they outlive the in-flight copies
        return (ticket.value, sd[0], oc[0], tn[0], st_[0])

    def playout_host_wait(self, ticket):
        """Block until the episode of ``ticket`` has its outputs in host memory;
        returns (outcomes or None, turns or None, stats)."""
        stuck = ctypes.c_int64(-1)
        native.check(native.lib().lx_playout_host_wait(self.handle, ticket[0],
                                                       ctypes.byref(stuck)), stuck.value)
        return ticket[2], ticket[3], ticket[4]

    def with_seeds(self, state, seeds):
        """Copy of ``state`` whose rows draw from new RNG streams (the MCTS
        rollout re-keying, reference agents.py:229-233)."""
        out = state.copy()
        s = _u64_tensor(seeds, state.batch_size)
        native.check(native.lib().lx_set_seeds(self.handle, out.words.data_ptr(),
                                               state.batch_size, s.data_ptr(), self._stream()))
        return out

    # -- observation --
    def observe_device(self, state, player):
        state.sync()
        torch = _torch()
        B = state.batch_size
        planes = torch.empty((B, self.observation_planes, self.num_cells), dtype=torch.uint8,
                             device="cuda")
        native.check(native.lib().lx_observe(self.handle, state.words.data_ptr(), B,
                                             int(player), planes.data_ptr(), self._stream()))
        return planes.view(torch.bool)

    def observe(self, state, player):
        """(B, 2T+1, C) relative-owner planes + legal mask (compiler.py:611-626)."""
        state = self._device(state)
        return (self.observe_device(state, player).cpu().numpy(),
                self.legal_mask(state))

    # -- reference layout interchange --
    def ref_arrays(self, B, device, packed=False):
        """Reference-layout tensors for B envs; ``packed``: all of them views
        of one byte buffer (16-byte aligned fields), returned with it as
        (dict, buffer), so a whole export moves in one copy."""
        torch = _torch()
        C, L = self.num_cells, self.layout
        f = {"board_piece": ((B, C), torch.int8), "board_owner": ((B, C), torch.int8),
             "current_player": ((B,), torch.int8), "move_count": ((B,), torch.int32),
             "terminated": ((B,), torch.bool), "truncated": ((B,), torch.bool),
             "outcome": ((B,), torch.int8), "seeds": ((B,), torch.int64)}
        if L.scores:
            f["scores"] = ((B, 2), torch.int32)
        if L.passing:
            f["pass_streak"] = ((B,), torch.int16)
            f["pass_flags"] = ((B, 2), torch.bool)
        if L.must_move:
            f["must_move"] = ((B,), torch.int16)
        if L.last_action:
            f.update({"last_mover": ((B,), torch.int8), "last_kind": ((B,), torch.int8),
                      "last_source": ((B,), torch.int16), "last_dest": ((B,), torch.int16),
                      "last_dest_by_player": ((B, 2), torch.int16)})
        if L.transient_masks:
            for k in ("hopped_mask", "captured_mask", "promoted_mask"):
                f[k] = ((B, C), torch.bool)
        if L.connectivity:
            f["comp_labels"] = ((B, L.connectivity, C), torch.int16)
        if L.phase:
            f["phase"] = ((B,), torch.int8)
        if L.turn_pos:
            f["turn_pos"] = ((B,), torch.int8)
        if not packed:
            return {k: torch.empty(shape, dtype=dt, device=device) for k, (shape, dt) in f.items()}
        offs, total = {}, 0
        for k, (shape, dt) in f.items():
            n = int(np.prod(shape)) * torch.empty(0, dtype=dt).element_size()
            offs[k] = (total, n)
            total += (n + 15) // 16 * 16
        buf = torch.empty(max(total, 16), dtype=torch.uint8, device=device)
        out = {k: buf[o:o + n].view(f[k][1]).view(f[k][0]) for k, (o, n) in offs.items()}
        return out, buf

    def _ref_struct(self, tensors):
        return native.RefState(**{k: (tensors[k].data_ptr() if k in tensors else None)
                                  for k in native.REF_FIELDS})

    def export_device(self, state):
        """Device tensors in the reference GameState layout (lx_export)."""
        state.sync()
        t = self.ref_arrays(state.batch_size, "cuda")
        ref = self._ref_struct(t)
        native.check(native.lib().lx_export(self.handle, state.words.data_ptr(),
                                            state.batch_size, ctypes.byref(ref), self._stream()))
        return t

    def _export(self, state):
        """Host numpy arrays of every reference field: one lx_export into one
        packed device buffer, one device-to-host copy, numpy views into it."""
        state.sync()
        t, buf = self.ref_arrays(state.batch_size, "cuda", packed=True)
        native.check(native.lib().lx_export(self.handle, state.words.data_ptr(),
                                            state.batch_size, ctypes.byref(self._ref_struct(t)),
                                            self._stream()))
        # pinned destination (torch's caching host allocator recycles the
        # block once the previous export's arrays are gone): the copy runs at
        # PCIe speed instead of through the driver's pageable staging
        torch = _torch()
        host = torch.empty(buf.numel(), dtype=torch.uint8, pin_memory=True)
        host.copy_(buf)
        base = buf.data_ptr()
        out = {}
        for k, v in t.items():
            o = v.data_ptr() - base
            a = host[o:o + v.numel() * v.element_size()].view(v.dtype).view(v.shape).numpy()
            out[k] = a.view(np.uint64) if k == "seeds" else a
        return out

    def _import_into(self, state, arrays):
        """Overwrite ``state``'s device words from reference-layout numpy
        arrays (lx_import; Hex reach sets are rebuilt from the boards)."""
        torch = _torch()
        t = {}
        for k, v in arrays.items():
            if v is None or k not in native.REF_FIELDS:
                continue
            a = np.ascontiguousarray(v)
            if not a.flags.writeable:          # DeviceState's read-only planes
                a = a.copy()
            if a.dtype == np.uint64:
                a = a.view(np.int64)
            t[k] = torch.as_tensor(a).to("cuda")
        if int(t["move_count"].max()) >= 2 ** 31 or int(t["move_count"].min()) < 0:
            raise ValueError("move_count out of range")
        ref = self._ref_struct(t)
        native.check(native.lib().lx_import(self.handle, state.words.data_ptr(),
                                            state.batch_size, ctypes.byref(ref), self._stream()))
        torch.cuda.current_stream().synchronize()

    def from_reference(self, arrays):
        """DeviceState from reference-layout numpy arrays (lx_import)."""
        st = self.empty_state(len(arrays["seeds"]))
        self._import_into(st, arrays)
        return st


def _sync(state):
    """Write host-side edits of a DeviceState's reference fields back to the
    device before a device call reads it (see DeviceState)."""
    state.sync()
    return state


def _foreign_arrays(state):
    """Reference-layout numpy arrays of a state object that is not a
    DeviceState (e.g. a reference GameState built by GameState.repeat_rows /
    concat from DeviceState fields), or None for a DeviceState."""
    if isinstance(state, DeviceState):
        return None
    out = {}
    for k in FIELDS:
        v = getattr(state, k, None)
        if v is not None:
            out[k] = np.asarray(v)
    return out


def _u64_tensor(seeds, B):
    torch = _torch()
    if isinstance(seeds, torch.Tensor):
        return seeds.to(device="cuda", dtype=torch.int64).contiguous()
    a = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(B)).view(np.int64)
    return torch.as_tensor(a).to("cuda")


def compile_game(spec):
    return B200Game(spec)


def load_game(text):
    """Parse, validate, lower (+ NVRTC on first device use); raises on any
    failure like the reference (__init__.py:34-41 load_game): ParseError,
    InvalidShapeParam, ValidationFailure, CompileError."""
    from .errors import ValidationFailure
    from .geometry import Board
    from .validate import validate
    spec = parse_game(text)
    report = validate(spec, Board(spec.equipment.board))
    if not report.ok:
        raise ValidationFailure(report)
    return B200Game(spec, text)


def load_config_game(name):
    with open(os.path.join(GAMES_DIR, f"{name}.ldx")) as f:
        return load_game(f.read())


def precompile(names=("tic_tac_toe", "connect_four", "hex", "reversi", "pente"), prune=True):
    """NVRTC-compile the config games' cubins into the in-tree cache (no GPU)."""
    keys = {}
    for name in names:
        with open(os.path.join(GAMES_DIR, f"{name}.ldx")) as f:
            low = lower_game(parse_game(f.read()))
        keys[name] = native.compile_only(low.source, low.name)
    if prune:                       # cubins are <key>-g<group>.cubin
        live = set(keys.values())
        for fn in os.listdir(native.CACHE_DIR):
            if fn.endswith(".cubin") and fn.split("-g")[0] not in live:
                os.remove(os.path.join(native.CACHE_DIR, fn))
    return keys


__all__ = ["B200Game", "DeviceState", "ActionCodec", "StateLayout", "load_game",
           "load_config_game", "compile_game", "precompile", "CompileError", "EmptyMask"]
