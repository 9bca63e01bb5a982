import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
PLACEMENT_GAMES = ("tic_tac_toe", "connect_four", "hex", "reversi", "pente", "gomoku", "yavalath")
MOVEMENT_GAMES = ("english_draughts", "dai_hasami_shogi", "wolf_and_sheep", "gridworld")
GAMES = PLACEMENT_GAMES + MOVEMENT_GAMES          # the reference's 11-game corpus


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


def golden_arrays(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def golden_state(name, k):
    arr = golden_arrays(name)
    pre = f"p{k}_"
    return {key[len(pre):]: v for key, v in arr.items() if key.startswith(pre)}


def game_text(name):
    with open(os.path.join(ROOT, "paper_2506_22609_b200", "games", f"{name}.ldx")) as f:
        return f.read()


def ref_allocator(info):
    """B -> reference-layout numpy arrays for a lowered game's state layout
    (reference state.py:78-130)."""
    C, L = info["C"], info["layout"]

    def allocate(B):
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
            s["comp_labels"] = np.full((B, L["connectivity"], C), -1, np.int16)
        if L["transient_masks"]:
            for k in ("hopped_mask", "captured_mask", "promoted_mask"):
                s[k] = np.zeros((B, C), bool)
        if L["phase"]:
            s["phase"] = np.zeros(B, np.int8)
        if L["turn_pos"]:
            s["turn_pos"] = np.zeros(B, np.int8)
        return s
    return allocate


REF_FIELDS = ("board_piece", "board_owner", "current_player", "move_count", "terminated",
              "truncated", "outcome", "seeds", "scores", "pass_streak", "pass_flags",
              "must_move", "last_mover", "last_kind", "last_source", "last_dest",
              "last_dest_by_player", "hopped_mask", "captured_mask", "promoted_mask",
              "comp_labels", "phase", "turn_pos")


def ref_digest(arrays):
    """reference GameState.digest (state.py:180-188) of a dict of arrays."""
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    for name in REF_FIELDS:
        v = arrays.get(name)
        if v is not None:
            h.update(name.encode())
            h.update(np.ascontiguousarray(v).tobytes())
    return h.hexdigest()
