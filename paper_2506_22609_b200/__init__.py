"""B200-native backend for Ludax's batched game-simulation hot path.

    import paper_2506_22609_b200 as lx
    game = lx.load_game(open("games/connect_four.ldx").read())
    state = lx.engine.init(game, batch_size=1 << 20, seed=1)
    final = lx.engine.playout_random(game, seed=1, batch_size=1 << 20).final

Front end (DSL reader, geometry) on the host; rules lowered to sm_100a
kernels compiled with NVRTC behind the C-ABI in include/ludax_b200.h.
"""

from . import agents, engine, evaluation, rng  # noqa: F401
from .errors import (BoardLangError, CompileError, EmptyMask, IllegalAction,  # noqa: F401
                     ParseError, TerminalState, ValidationFailure)
from .validate import validate  # noqa: F401
from .game import (B200Game, DeviceState, compile_game, load_config_game,  # noqa: F401
                   load_game, precompile)
from .env import EnvState, LudaxEnvironment  # noqa: F401
from .syntax import parse_game  # noqa: F401

__version__ = "0.1.0"
