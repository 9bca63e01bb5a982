import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
GAMES = ("tic_tac_toe", "connect_four", "hex", "reversi", "pente", "gomoku", "yavalath")


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
