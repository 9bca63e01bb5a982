"""Generality of the lowering on programs from the reference's own random
game generator (generator.sample_game, four corpora: sampler seeds 7, 11, 23, 31,
tests/golden/fuzz.json made by oracle/gen_golden.py --fuzz): every program the reference plays must be
lowered bit-exactly -- final-state digest and env-step count of seeded
playouts -- or rejected with CompileError (no silent divergence)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, ref_allocator, ref_digest
from paper_2506_22609_b200 import lowering, rng, syntax
from paper_2506_22609_b200.errors import CompileError

with open(os.path.join(GOLDEN, "fuzz.json")) as f:
    FUZZ = json.load(f)
PROGRAMS = FUZZ["programs"]
MAX_UNSUPPORTED = 0


def lowered(prog):
    try:
        return lowering.lower_game(syntax.parse_game(prog["text"]))
    except CompileError:
        return None


def test_fuzz_corpus_coverage():
    unsupported = [p["index"] for p in PROGRAMS if lowered(p) is None]
    assert len(unsupported) <= MAX_UNSUPPORTED, unsupported
    assert len(PROGRAMS) >= 570


@pytest.mark.parametrize("prog", PROGRAMS[::16],
                         ids=lambda p: f"s{p.get('sampler', [7])[0]}-{p['index']}")
def test_fuzz_hostsim_matches_reference(prog):
    from hostsim.hostsim import HostGame
    low = lowered(prog)
    if low is None:
        pytest.skip("not lowered (CompileError)")
    hg = HostGame(low)
    for run in prog["runs"]:
        got, steps = hg.playout(rng.spawn_seeds(run["seed"], FUZZ["batch"]),
                                max_turns=FUZZ["max_turns"], layout_arrays=ref_allocator(low.info))
        assert ref_digest(got) == run["digest"]
        assert steps == run["turns"]


def _fuzz_part(default_stride):
    """LX_FUZZ_ALL=1: the whole corpus; LX_FUZZ_ALL=k/n: programs k, k+n, ...
    (the corpus in n GPU calls); else a stride sample."""
    spec = os.environ.get("LX_FUZZ_ALL")
    if not spec:
        return PROGRAMS[::default_stride]
    if "/" in spec:
        k, n = (int(x) for x in spec.split("/"))
        return PROGRAMS[k::n]
    return PROGRAMS


@pytest.mark.gpu
def test_fuzz_device_matches_reference():
    """A stride-30 sample (NVRTC compiles each program in ~7 s; the whole
    corpus passed on a B200 in round 1: LX_FUZZ_ALL=1 runs it)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_22609_b200 as lx
    part = _fuzz_part(30)
    checked = 0
    for prog in part:
        if lowered(prog) is None:
            continue
        g = lx.load_game(prog["text"])
        for run in prog["runs"]:
            po = lx.engine.playout_random(g, seed=run["seed"], batch_size=FUZZ["batch"],
                                          max_turns=FUZZ["max_turns"])
            assert po.final.digest() == run["digest"], prog["index"]
            assert int(np.asarray(po.turns_taken).sum()) == run["turns"], prog["index"]
        checked += 1
    assert checked == len(part)


with open(os.path.join(GOLDEN, "fuzz_masks.json")) as f:
    MASKS = json.load(f)
_TEXT = {(tuple(p.get("sampler") or [7, 5]), p["index"]): p["text"] for p in PROGRAMS}


def _mask_hash(row):
    import hashlib
    return hashlib.blake2b(np.packbits(np.asarray(row, dtype=bool)).tobytes(),
                           digest_size=8).hexdigest()


@pytest.mark.parametrize("rec", MASKS["programs"][::3],
                         ids=lambda r: f"s{(r.get('sampler') or [7])[0]}-{r['index']}")
def test_fuzz_hostsim_masks_match_reference(rec):
    """Per-ply legal masks and sampled actions (reference fuzz_masks.json)."""
    from hostsim.hostsim import HostGame
    text = _TEXT[(tuple(rec.get("sampler") or [7, 5]), rec["index"])]
    hg = HostGame(lowering.lower_game(syntax.parse_game(text)))
    seeds = rng.spawn_seeds(3, 4)
    for i in range(4):
        want = rec["rows"][i]
        m, a = hg.masks(int(seeds[i]), max_plies=60)
        assert len(a) >= len(want)
        for t, (h, act) in enumerate(want):
            assert _mask_hash(m[t]) == h, (i, t)
            assert int(a[t]) == act, (i, t)


@pytest.mark.gpu
def test_fuzz_device_masks_match_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_22609_b200 as lx
    every = 1 if os.environ.get("LX_FUZZ_ALL") else 6
    for rec in MASKS["programs"][::every]:
        g = lx.load_game(_TEXT[(tuple(rec.get("sampler") or [7, 5]), rec["index"])])
        st = g.init(4, seed=3)
        t = 0
        while t < 60 and not st.terminated.all():
            m = g.legal_mask(st)
            a = lx.engine.random_actions(g, st)
            live = ~st.terminated
            if (a[live] < 0).any():
                break
            for i in np.nonzero(live)[0]:
                assert [_mask_hash(m[i]), int(a[i])] == rec["rows"][i][t], (rec["index"], i, t)
            g.step_into(st, a, rows=live, verify=True)
            t += 1
        assert st.digest() == rec["digest"], rec["index"]
