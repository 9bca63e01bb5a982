"""The lowered rules (the exact code the sm_100a kernels run), compiled for the
host by tests/hostsim, against the oracle -- catches lowering bugs on CPU."""
import numpy as np
import pytest

from conftest import GAMES, game_text
from hostsim.hostsim import HostGame
from oracle import oracle as O
from paper_2506_22609_b200 import lowering, rng, syntax

B = {"tic_tac_toe": 4096, "connect_four": 2048, "hex": 512, "reversi": 1024, "pente": 128,
     "gomoku": 256, "yavalath": 1024, "english_draughts": 256, "dai_hasami_shogi": 128,
     "wolf_and_sheep": 1024, "gridworld": 4096}


@pytest.fixture(scope="module", params=GAMES)
def pair(request):
    name = request.param
    low = lowering.lower_game(syntax.parse_game(game_text(name)))
    return name, HostGame(low), O.OracleGame(name)


def test_hostsim_playouts_equal_oracle(pair):
    name, hg, og = pair
    seeds = rng.spawn_seeds(31337, B[name])
    got, steps = hg.playout(seeds, layout_arrays=og.allocate)
    want, wsteps = og.playout(state=og.init(B[name], seeds=seeds))
    assert steps == wsteps
    for f, v in want.items():
        assert np.array_equal(got[f], v), (name, f)
    assert O.digest(got) == O.digest(want)


def test_state_layout_matches_lowering_info(pair):
    """lx::Layout (device pack/unpack) and the lowering's word count agree."""
    name, hg, og = pair
    assert hg.layout() == (hg.info["nwords"], hg.info["nq"]), name


def test_hostsim_masks_equal_oracle(pair):
    name, hg, og = pair
    for seed in rng.spawn_seeds(5, 6):
        masks, actions = hg.masks(int(seed))
        st = og.init(1, seeds=np.array([seed], dtype=np.uint64))
        for t in range(len(actions)):
            m, _ = og.legal_mask(st)
            assert np.array_equal(masks[t], m[0]), (name, t)
            og.step_into(st, actions[t:t + 1], verify=True)
