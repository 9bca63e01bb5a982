"""cProfile of evaluation.evaluate_game on a corpus game (device path)."""
import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2506_22609_b200 as lx  # noqa: E402
from paper_2506_22609_b200 import evaluation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tic_tac_toe"
text = open(os.path.join(os.path.dirname(lx.__file__), "games", f"{name}.ldx")).read()
lx.load_game(text).native                     # NVRTC / module load outside the profile
cfg = evaluation.EvalConfig(matches=100)
pr = cProfile.Profile()
pr.enable()
evaluation.evaluate_game(text, cfg)
pr.disable()
out = io.StringIO()
pstats.Stats(pr, stream=out).sort_stats("cumtime").print_stats(25)
print(out.getvalue()[:5000])
