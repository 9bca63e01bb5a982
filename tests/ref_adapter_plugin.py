"""pytest plugin -- TEST INFRASTRUCTURE: runs the reference's own test files
(staged by __graft_entry__.stage_reference into baseline/_ref/ref_tests)
with ``boardlang.load_game`` swapped for this backend's ``load_game``, so
their ``compiled(name)`` fixtures hand the reference's engine / evaluation
code a B200Game (the reference's loops and tests drive the
adapter).  Loaded with ``-p ref_adapter_plugin``."""
import boardlang

import paper_2506_22609_b200 as lx

boardlang.load_game = lx.load_game

# the binding raises the reference's exception types: status
# codes map onto boardlang.errors classes instead of this package's own
from boardlang import errors as _ref_errors  # noqa: E402

for _n in ("IllegalAction", "TerminalState", "EmptyMask"):
    setattr(lx.errors, _n, getattr(_ref_errors, _n))
