"""ctypes wrapper of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  States are dicts of numpy arrays in the reference GameState
field layout (reference: pkg/src/boardlang/state.py:34-130); ``digest``
reproduces GameState.digest (state.py:180-188) byte for byte, so oracle,
device export and reference fixtures are compared on the same key.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libludax_oracle.so")

FIELDS = ("board_piece", "board_owner", "current_player", "move_count",
          "terminated", "truncated", "outcome", "seeds", "scores", "pass_streak",
          "pass_flags", "must_move", "last_mover", "last_kind", "last_source",
          "last_dest", "last_dest_by_player", "hopped_mask", "captured_mask",
          "promoted_mask", "comp_labels", "phase", "turn_pos")

GAMES = ("tic_tac_toe", "connect_four", "hex", "reversi", "pente", "gomoku", "yavalath",
         "english_draughts", "dai_hasami_shogi", "wolf_and_sheep", "gridworld")


class _SoA(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in (
        "board_piece", "board_owner", "current_player", "move_count", "terminated",
        "truncated", "outcome", "seeds", "scores", "pass_streak", "pass_flags",
        "last_mover", "last_kind", "last_source", "last_dest", "last_dest_by_player",
        "comp_labels", "phase", "must_move")]


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or (
                os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "ludax_oracle.c"))):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.orc_game_new.restype = vp
        L.orc_game_new.argtypes = [ctypes.c_char_p]
        for f in ("orc_num_cells", "orc_num_actions", "orc_layout", "orc_mechanics"):
            getattr(L, f).restype = i32
            getattr(L, f).argtypes = [vp]
        L.orc_init.argtypes = [vp, ctypes.POINTER(_SoA), i64, vp]
        L.orc_spawn_seeds.argtypes = [ctypes.c_uint64, i64, i64, vp]
        L.orc_hash_key3.restype = ctypes.c_uint64
        L.orc_hash_key3.argtypes = [ctypes.c_uint64] * 3
        L.orc_legal.argtypes = [vp, ctypes.POINTER(_SoA), i64, vp, vp]
        L.orc_sample.argtypes = [vp, ctypes.POINTER(_SoA), i64, vp, vp]
        L.orc_step.restype = i32
        L.orc_step.argtypes = [vp, ctypes.POINTER(_SoA), i64, vp, vp, i32, ctypes.POINTER(i64)]
        L.orc_playout.restype = i64
        L.orc_playout.argtypes = [vp, ctypes.POINTER(_SoA), i64, i32, i32, ctypes.POINTER(i64)]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleGame:
    """One config game in the oracle; states are dicts of numpy arrays."""

    def __init__(self, name):
        self.name = name
        self.h = lib().orc_game_new(name.encode())
        if not self.h:
            raise KeyError(f"oracle has no game {name!r}")
        self.C = lib().orc_num_cells(self.h)
        self.A = lib().orc_num_actions(self.h)
        lay = lib().orc_layout(self.h)
        self.layout = {"scores": bool(lay & 1), "passing": bool(lay & 2),
                       "last_action": bool(lay & 4), "connectivity": bool(lay & 8),
                       "phase": bool(lay & 16), "must_move": bool(lay & 32)}
        self.mechanics = lib().orc_mechanics(self.h)
        self.pass_index = self.C if (self.mechanics == 0 and self.A > self.C) else None

    def allocate(self, B):
        C, L = self.C, self.layout
        s = {"board_piece": np.full((B, C), -1, np.int8),
             "board_owner": np.full((B, C), -1, np.int8),
             "current_player": np.zeros(B, np.int8), "move_count": np.zeros(B, np.int32),
             "terminated": np.zeros(B, bool), "truncated": np.zeros(B, bool),
             "outcome": np.full(B, -1, np.int8), "seeds": np.zeros(B, np.uint64)}
        if L["scores"]:
            s["scores"] = np.zeros((B, 2), np.int32)
        if L["passing"]:
            s["pass_streak"] = np.zeros(B, np.int16)
            s["pass_flags"] = np.zeros((B, 2), bool)
        if L["must_move"]:
            s["must_move"] = np.full(B, -1, np.int16)
        if L["last_action"]:
            s["last_mover"] = np.full(B, -1, np.int8)
            s["last_kind"] = np.full(B, -1, np.int8)
            s["last_source"] = np.full(B, -1, np.int16)
            s["last_dest"] = np.full(B, -1, np.int16)
            s["last_dest_by_player"] = np.full((B, 2), -1, np.int16)
        if L["connectivity"]:
            s["comp_labels"] = np.full((B, 1, C), -1, np.int16)
        if L["phase"]:
            s["phase"] = np.zeros(B, np.int8)
        return s

    @staticmethod
    def _soa(s):
        return _SoA(**{f: _ptr(s.get(f)) for f, _ in _SoA._fields_})

    def init(self, batch_size=1, seed=0, seeds=None):
        if seeds is None:
            seeds = spawn_seeds(seed, batch_size)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64).reshape(-1)
        s = self.allocate(len(seeds))
        lib().orc_init(self.h, ctypes.byref(self._soa(s)), len(seeds), _ptr(seeds))
        return s

    def legal_mask(self, s):
        B = len(s["seeds"])
        mask = np.zeros((B, self.A), np.uint8)
        counts = np.zeros(B, np.int64)
        lib().orc_legal(self.h, ctypes.byref(self._soa(s)), B, _ptr(mask), _ptr(counts))
        return mask.astype(bool), counts

    def sample_actions(self, s, u=None):
        B = len(s["seeds"])
        out = np.zeros(B, np.int64)
        if u is not None:
            u = np.ascontiguousarray(u, dtype=np.float64)
        lib().orc_sample(self.h, ctypes.byref(self._soa(s)), B, _ptr(u), _ptr(out))
        return out

    def step_into(self, s, actions, rows=None, verify=True):
        B = len(s["seeds"])
        actions = np.ascontiguousarray(np.broadcast_to(actions, (B,)), dtype=np.int64)
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.uint8)
        bad = ctypes.c_int64(-1)
        st = lib().orc_step(self.h, ctypes.byref(self._soa(s)), B, _ptr(actions), _ptr(r),
                            int(verify), ctypes.byref(bad))
        return st, bad.value

    def playout(self, batch_size=1, seed=0, seeds=None, max_turns=200, threads=1, state=None):
        """engine.playout_random equivalent; returns (final state, env steps)."""
        s = state if state is not None else self.init(batch_size, seed, seeds)
        stuck = ctypes.c_int64(-1)
        steps = lib().orc_playout(self.h, ctypes.byref(self._soa(s)), len(s["seeds"]),
                                  max_turns, threads, ctypes.byref(stuck))
        if stuck.value >= 0:
            raise RuntimeError(f"oracle: row {stuck.value} has no legal action")
        return s, steps


def spawn_seeds(seed, count, first=0):
    out = np.zeros(count, np.uint64)
    lib().orc_spawn_seeds(int(seed) & (2**64 - 1), first, count, _ptr(out))
    return out


def hash_key3(a, b, c):
    return int(lib().orc_hash_key3(a, b, c))


def digest(state):
    """Byte-identical to the reference GameState.digest (state.py:180-188)."""
    h = hashlib.blake2b(digest_size=16)
    for name in FIELDS:
        v = state.get(name)
        if v is not None:
            h.update(name.encode())
            h.update(np.ascontiguousarray(v).tobytes())
    return h.hexdigest()
