"""Movement / gridworld lowering on the CPU: the generated
rules compiled for the host (tests/hostsim) against fixtures produced by the
reference itself (oracle/gen_golden.py): seeded random playouts, per-ply
legal masks, and the transcripts of the reference's own tests
(test_acceptance.py:148-178, test_engine.py:159-196, test_compiler.py:198-204)."""
import numpy as np
import pytest

from conftest import (MOVEMENT_GAMES, game_text, golden_arrays, golden_state, ref_allocator,
                      ref_digest)
from hostsim.hostsim import HostGame
from paper_2506_22609_b200 import lowering, rng, syntax


def host_game(text):
    low = lowering.lower_game(syntax.parse_game(text))
    return low, HostGame(low)


@pytest.fixture(scope="module", params=MOVEMENT_GAMES)
def mgame(request):
    name = request.param
    low, hg = host_game(game_text(name))
    return name, low, hg


def test_movement_playouts_match_reference(mgame, golden_meta):
    name, low, hg = mgame
    for k, po in enumerate(golden_meta["games"][name]["playouts"]):
        seeds = rng.spawn_seeds(po["seed"], po["batch"])
        got, steps = hg.playout(seeds, layout_arrays=ref_allocator(low.info))
        want = golden_state(name, k)
        assert set(got) == set(want), (name, sorted(set(got) ^ set(want)))
        for f, v in want.items():
            assert np.array_equal(got[f], v), (name, k, f)
        assert ref_digest(got) == po["digest"]
        assert steps == po["turns"]


def test_movement_trajectory_masks(mgame, golden_meta):
    name, low, hg = mgame
    arr = golden_arrays(name)
    A = golden_meta["games"][name]["traj_mask_width"]
    assert A == low.info["A"]
    masks = np.unpackbits(arr["traj_masks"], axis=-1)[..., :A].astype(bool)   # (T, 4, A)
    actions = arr["traj_actions"]
    seeds = rng.spawn_seeds(3, 4)
    for i in range(4):
        m, a = hg.masks(int(seeds[i]), max_plies=len(actions))
        T = len(a)
        assert np.array_equal(m, masks[:T, i]), (name, i)
        assert np.array_equal(a, actions[:T, i]), (name, i)
        if T < len(actions):
            assert (actions[T:, i] == -1).all()


def test_draughts_forced_capture(golden_meta):
    kat = golden_meta["kat"]["draughts_forced"]
    low, hg = host_game(game_text("english_draughts"))
    acts = kat["actions"] + [17 * 64 + 35]
    arrays, masks, ok, t = hg.transcript(acts[:3], layout_arrays=ref_allocator(low.info))
    assert ok.all() and t == 3
    assert np.nonzero(masks[3])[0].tolist() == kat["legal"]
    assert ref_digest(arrays) == kat["digest"]
    arrays, masks, ok, t = hg.transcript(acts, layout_arrays=ref_allocator(low.info))
    assert ok.all() and t == 4
    assert ref_digest(arrays) == kat["after_capture"]["digest"]
    assert int(arrays["current_player"][0]) == kat["after_capture"]["current_player"] == 0


def test_draughts_double_jump_drill(golden_meta):
    kat = golden_meta["kat"]["draughts_drill"]
    text = game_text("english_draughts")
    for a, b in kat["text_replace"]:
        text = text.replace(a, b)
    low, hg = host_game(text)
    alloc = ref_allocator(low.info)
    _, masks, ok, t = hg.transcript([], layout_arrays=alloc)
    assert np.nonzero(masks[0])[0].tolist() == kat["start_legal"]
    arrays, masks, ok, t = hg.transcript([36 * 64 + 18], layout_arrays=alloc)
    assert ok.all()
    assert int(arrays["current_player"][0]) == kat["after1"]["current_player"]
    assert int(arrays["must_move"][0]) == kat["after1"]["must_move"] == 18
    assert np.nonzero(masks[1])[0].tolist() == kat["after1"]["legal"]
    assert ref_digest(arrays) == kat["after1"]["digest"]
    arrays, masks, ok, t = hg.transcript([36 * 64 + 18, 18 * 64 + 0], layout_arrays=alloc)
    assert ok.all()
    assert int(arrays["board_piece"][0, 0]) == kat["after2"]["piece0"] == 1
    assert int(arrays["current_player"][0]) == kat["after2"]["current_player"]
    assert ref_digest(arrays) == kat["after2"]["digest"]


def test_draughts_priority_rejects_step_when_hop_exists():
    low, hg = host_game(game_text("english_draughts"))
    # after the forced-capture opening a step is in no mask and is illegal
    _, masks, ok, t = hg.transcript([44 * 64 + 35, 21 * 64 + 30, 35 * 64 + 26, 17 * 64 + 26],
                                    layout_arrays=ref_allocator(low.info))
    assert t == 3 and not ok[3]


def test_gridworld_transcript(golden_meta):
    kat = golden_meta["kat"]["gridworld"]
    low, hg = host_game(game_text("gridworld"))
    assert low.info["grid_directions"] == kat["directions"]
    _, masks, ok, t = hg.transcript([], layout_arrays=ref_allocator(low.info))
    assert np.nonzero(masks[0])[0].tolist() == kat["initial_legal"]
    arrays, masks, ok, t = hg.transcript(kat["right_down"]["actions"],
                                         layout_arrays=ref_allocator(low.info))
    assert ok.all()
    assert ref_digest(arrays) == kat["right_down"]["digest"]
    assert int(arrays["outcome"][0]) == kat["right_down"]["outcome"] == 2
