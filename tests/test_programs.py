"""Test programs that each pin one property the corpus games never reach
(tests/programs/*.ldx) against the reference's own playouts
(tests/golden/programs.json, oracle/gen_golden.py --programs).

big_score.ldx: scores beyond int16 (up to ~10^5).  The host emulation
round-trips the packed device state every ply, so the CPU test pins the
32-bit score words of the HBM layout; the GPU tests run the per-ply stepped
path (lx_step, state stored every ply), the PGX env path and the fused
rollout."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, has_gpu, ref_allocator
from hostsim.hostsim import HostGame
from oracle import oracle as O
from paper_2506_22609_b200 import lowering, rng, syntax

PROGRAMS = json.load(open(os.path.join(GOLDEN, "programs.json")))


def _text(name):
    return open(os.path.join(ROOT, "tests", "programs", f"{name}.ldx")).read()


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_program_hostsim_matches_reference(name):
    low = lowering.lower_game(syntax.parse_game(_text(name)))
    hg = HostGame(low)
    for run in PROGRAMS[name]:
        seeds = rng.spawn_seeds(run["seed"], run["batch"])
        got, _ = hg.playout(seeds, layout_arrays=ref_allocator(low.info))
        assert O.digest(got) == run["digest"], (name, run["seed"])
        if run["scores"] is not None:
            assert got["scores"].tolist() == run["scores"]


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_program_device_paths_match_reference(name):
    import paper_2506_22609_b200 as lx
    g = lx.load_game(_text(name))
    for run in PROGRAMS[name]:
        B, seed = run["batch"], run["seed"]
        fused = lx.engine.playout_random(g, seed=seed, batch_size=B).final
        stepped = lx.engine.playout_random(g, seed=seed, batch_size=B, record=True).final
        assert fused.digest() == run["digest"]
        assert stepped.digest() == run["digest"]
        env = lx.LudaxEnvironment(g, max_steps=200)
        st = env.init(seed=seed, batch_size=B)
        while not bool(st.terminated.all()):
            st = env.step_(st, env.RANDOM)
        assert st.game_state.digest() == run["digest"]
        if run["scores"] is not None:
            assert np.array_equal(st.game_state.scores, np.array(run["scores"], np.int32))
