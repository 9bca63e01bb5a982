"""The reference's own loops and tests driving this backend.

The unmodified reference (baseline/_ref, installed by build() from
/root/reference) is imported, and its ``evaluation._run_episode``
(evaluation.py:197-211) and ``engine.playout_random`` (engine.py:123-163)
run with a B200Game in place of its CompiledGame; step counts, final-state
digests and recorded trajectories must equal the reference's own run.
Its engine test file (tests/test_engine.py) then runs with its compiled()
fixture swapped to paper_2506_22609_b200.load_game (tests/ref_adapter_plugin.py).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, game_text

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "boardlang")):
    pytest.skip("baseline/_ref is not staged (build() installs the reference there)",
                allow_module_level=True)
sys.path.insert(0, REF)

import boardlang  # noqa: E402
from boardlang import engine as ref_engine, evaluation as ref_eval, rng as ref_rng  # noqa: E402

import paper_2506_22609_b200 as lx  # noqa: E402

_REF_LOAD = boardlang.load_game
CASES = [("tic_tac_toe", 1024), ("connect_four", 512), ("hex", 128), ("reversi", 256),
         ("pente", 64), ("english_draughts", 64), ("yavalath", 128), ("gridworld", 256)]


@pytest.mark.parametrize("name,B", CASES)
def test_reference_run_episode_drives_adapter(name, B):
    ours, ref = lx.load_config_game(name), _REF_LOAD(game_text(name))
    for e in (0, 10_000):
        seed = ref_rng.hash_key(np.uint64(0), np.uint64(B), np.uint64(e))
        want, _ = ref_eval._run_episode(ref, B, seed, 200)
        got, _ = ref_eval._run_episode(ours, B, seed, 200)      # reference loop, our kernels
        fused, _ = lx.evaluation._run_episode(ours, B, seed, 200)
        assert got == want == fused, (name, e)


@pytest.mark.parametrize("name,B", CASES)
def test_reference_playout_random_drives_adapter(name, B):
    ours, ref = lx.load_config_game(name), _REF_LOAD(game_text(name))
    B = min(B, 64)
    want = ref_engine.playout_random(ref, seed=13, batch_size=B, max_turns=200, record=True)
    got = ref_engine.playout_random(ours, seed=13, batch_size=B, max_turns=200, record=True)
    assert got.final.digest() == want.final.digest()
    assert [got.to_jsonl(i) for i in range(0, B, 7)] == [want.to_jsonl(i) for i in range(0, B, 7)]
    assert np.array_equal(got.turns_taken, want.turns_taken)
    # and the backend's own fused path agrees with both
    assert lx.engine.playout_random(ours, seed=13, batch_size=B).final.digest() == \
        want.final.digest()


REF_FILES = {
    # the reference's engine tests: all of them
    "test_engine.py": None,
    # acceptance tests that exercise the engine path (the GAVEL / MCTS /
    # generator ones drive the reference's own agents and CLI;
    # draughts_transcript_and_priority reads CompiledGame internals,
    # `phases[0].mechanics`, that are not part of the API)
    "test_acceptance.py": "corpus or exhaustive or hex_has_no_draws or reversi_integrity or "
                          "batch_equals_sequential or throughput_scaling",
}


@pytest.mark.parametrize("fname", sorted(REF_FILES))
def test_reference_test_file_over_adapter(fname):
    tests = os.path.join(REF, "ref_tests")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, os.path.join(ROOT, "tests"), ROOT,
                                                      tests]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_adapter_plugin",
           "-p", "no:cacheprovider", "-rf", os.path.join(tests, fname)]
    if REF_FILES[fname]:
        cmd += ["-k", REF_FILES[fname]]
    p = subprocess.run(cmd, cwd=tests, env=env, capture_output=True, text=True, timeout=1500)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"ref_{fname[:-3]}_over_adapter.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    assert p.returncode == 0, p.stdout[-4000:]
