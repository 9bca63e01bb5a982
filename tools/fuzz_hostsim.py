"""Whole generated-program corpus (tests/golden/fuzz.json) through the host
emulation of the lowered rules (tests/hostsim): digest + step count of every
seeded playout vs the reference's.  CPU only; ~5-10 minutes.

    python tools/fuzz_hostsim.py [--stride 1]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import ref_allocator, ref_digest  # noqa: E402
from hostsim.hostsim import HostGame  # noqa: E402
from paper_2506_22609_b200 import lowering, rng, syntax  # noqa: E402
from paper_2506_22609_b200.errors import CompileError  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--stride", type=int, default=1)
a = p.parse_args()
F = json.load(open(os.path.join(ROOT, "tests", "golden", "fuzz.json")))
ok, bad, unsupported = 0, [], []
t0 = time.time()
for prog in F["programs"][::a.stride]:
    try:
        low = lowering.lower_game(syntax.parse_game(prog["text"]))
    except CompileError:
        unsupported.append(prog["index"])
        continue
    hg = HostGame(low)
    good = True
    for run in prog["runs"]:
        got, steps = hg.playout(rng.spawn_seeds(run["seed"], F["batch"]), max_turns=F["max_turns"],
                                layout_arrays=ref_allocator(low.info))
        good &= ref_digest(got) == run["digest"] and steps == run["turns"]
    if good:
        ok += 1
    else:
        bad.append((prog.get("sampler"), prog["index"]))
print(json.dumps({"programs": len(F["programs"][::a.stride]), "bit_exact": ok, "mismatch": bad,
                  "unsupported": unsupported, "seconds": round(time.time() - t0, 1)}))
