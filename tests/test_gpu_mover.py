"""Legality for a non-current mover (the reference's `mover=` argument of
legal_mask / legal_counts / sample_actions, compiler.py:394-446) against the
reference's own answers on its own states (tests/golden/mover.npz, written by
oracle/gen_golden.py --mover): states imported through lx_import, mover
flipped on odd rows."""
import os

import numpy as np
import pytest

from conftest import GAMES, GOLDEN

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402
from oracle import oracle as O  # noqa: E402

FIX = dict(np.load(os.path.join(GOLDEN, "mover.npz")))


def _snapshots(name):
    out = {}
    for key, v in FIX.items():
        g, k, field = key.split("__")
        if g == name:
            out.setdefault(int(k), {})[field] = v
    return out


@pytest.mark.parametrize("name", GAMES)
def test_mover_override_matches_reference(name):
    g = lx.load_config_game(name)
    snaps = _snapshots(name)
    assert snaps
    for k, fx in sorted(snaps.items()):
        arrays = {f: fx[f] for f in fx if f not in ("mover", "u", "mask", "counts", "sampled")}
        st = g.from_reference(arrays)
        mover = fx["mover"]
        assert np.array_equal(g.legal_mask(st, mover=mover), fx["mask"]), (name, k)
        assert np.array_equal(g.legal_counts(st, mover=mover), fx["counts"]), (name, k)
        assert np.array_equal(g.sample_actions(st, fx["u"], mover=mover), fx["sampled"]), (name, k)
        # the override changes nothing stored: current-mover answers are unchanged
        cur = arrays["current_player"]
        assert np.array_equal(g.legal_mask(st, mover=cur), g.legal_mask(st))
        assert st.digest() == O.digest(arrays)                  # import -> export round trip
