"""Host front end: DSL reader, geometry, lowering (no GPU needed)."""
import dataclasses

import numpy as np
import pytest

from conftest import GAMES, game_text
from paper_2506_22609_b200 import geometry, lowering, nodes, syntax
from paper_2506_22609_b200.errors import CompileError, ParseError


def norm(x):
    if dataclasses.is_dataclass(x):
        return [type(x).__name__] + [[f.name, norm(getattr(x, f.name))]
                                     for f in dataclasses.fields(x)]
    if isinstance(x, tuple):
        return [norm(i) for i in x]
    return x


def jsonable(x):
    import json
    return json.loads(json.dumps(x))


@pytest.mark.parametrize("name", GAMES)
def test_parser_matches_reference_ast(name, golden_meta):
    """Same AST as the reference parser (dump made by oracle/gen_golden.py)."""
    spec = syntax.parse_game(game_text(name))
    assert jsonable(norm(spec)) == golden_meta["games"][name]["ast"]


@pytest.mark.parametrize("name", GAMES)
def test_layout_and_codec_match_reference(name, golden_meta):
    d = golden_meta["games"][name]["describe"]
    low = lowering.lower_game(syntax.parse_game(game_text(name)))
    assert low.info["C"] == d["num_cells"]
    assert low.info["A"] == d["action_space"]["size"]
    assert (low.info["pass_index"] >= 0) == d["action_space"]["has_pass"]
    assert low.info["codec"] == d["action_space"]["kind"]
    assert low.info["observation_planes"] == d["observation_planes"]
    L = low.info["layout"]
    ref = d["state_layout"]
    for k_ref, k in (("scores", "scores"), ("passing", "passing"), ("must_move", "must_move"),
                     ("last_action", "last_action"), ("transient_masks", "transient_masks"),
                     ("connectivity_plans", "connectivity"), ("phase_index", "phase"),
                     ("turn_position", "turn_pos")):
        assert L[k] == ref[k_ref], k


@pytest.mark.parametrize("bad", [
    "(game", "(game \"x\" (players 2))", "(game \"x\" (players 2) (equipment (board (square 0))))",
    "(game \"x\" (players 2) (equipment (board (square 3)) (pieces (\"s\" both))) "
    "(rules (play (repeat (P1 P2) (place \"s\" (destination (bogus))))) (end (if (full_board) (draw)))))",
])
def test_parse_errors(bad):
    with pytest.raises(ParseError):
        syntax.parse_game(bad)


def test_token_deletion_fuzz_never_crashes():
    """Dropping any single token either parses or raises ParseError
    (reference tests/test_parser.py:164)."""
    text = game_text("reversi")
    toks = [m.group() for m in syntax._TOKEN.finditer(text)]
    for i in range(0, len(toks), 3):
        try:
            syntax.parse_game("".join(toks[:i] + toks[i + 1:]))
        except ParseError:
            pass


@pytest.mark.parametrize("shape", [("square", 3, 3), ("rectangle", 6, 7),
                                   ("hex_rectangle", 11, 11), ("square", 19, 19),
                                   ("hexagon", 5, 5)])
def test_neighbor_symmetry(shape):
    b = geometry.Board(nodes.BoardShape(*shape))
    for d in b.directions:
        inv = b.neighbors[geometry.OPPOSITE[d]]
        for c in range(b.num_cells):
            n = b.neighbors[d][c]
            if n != b.sentinel:
                assert inv[n] == c


def test_line_windows_counts():
    b = geometry.Board(nodes.BoardShape("rectangle", 6, 7))
    assert len(b.line_windows(4, "any")) == 69
    b = geometry.Board(nodes.BoardShape("square", 19, 19))
    assert len(b.line_windows(5, "any")) == 1020
    b = geometry.Board(nodes.BoardShape("square", 3, 3))
    assert len(b.line_windows(3, "any")) == 8


@pytest.mark.parametrize("name", GAMES)
def test_lowering_shift_proof_and_source(name):
    gl = lowering.GameLowering(syntax.parse_game(game_text(name)))
    for d in gl.board.directions:
        S = gl._shift[d]
        nt = gl.board.neighbors[d]
        for x in range(gl.C):
            if nt[x] != gl.C:
                assert gl.bit_of[nt[x]] == gl.bit_of[x] + S
    src = gl.lower().source
    assert "struct Game" in src and '#include "lx_kernels.cuh"' in src


def test_lowering_words_bit_order():
    m = np.zeros(42, dtype=bool)
    m[[0, 31, 32, 41]] = True
    w = lowering._words(m, 2)
    assert w == ((1 << 0) | (1 << 31), (1 << 0) | (1 << 9))


@pytest.mark.parametrize("text,what", [
    ("""(game "AX" (players 2) (equipment (board (square 8)) (pieces ("s" both)))
        (rules (play (repeat (P1 P2) (place "s" (destination (empty)))))
        (end (if (and (mover_is P1) (line "s" 4 exact:true exclude:((row 0)))) (mover win))
             (if (full_board) (draw)))))""", "exact anchored line with exclude"),
    ("""(game "Two" (players 2) (equipment (board (square 5)) (pieces ("s" both)))
        (rules (play (repeat (P1 P2) (place "s" (destination (empty)))))
        (end (if (connected "s" ((edge top) (edge bottom)) direction:orthogonal) (mover win))
             (if (connected "s" ((edge left) (edge right))) (mover win)))))""",
     "two connectivity plans"),
    ("""(game "Tri" (players 2) (equipment (board (square 5)) (pieces ("s" both)))
        (rules (play (repeat (P1 P2) (place "s" (destination (empty)))))
        (end (if (connected "s" ((edge top) (edge bottom) (edge left))) (mover win)))))""",
     "three-target connected"),
])
def test_formerly_unsupported_constructs_lower(text, what):
    low = lowering.lower_game(syntax.parse_game(text))
    assert "struct Game" in low.source, what


def test_reference_unsupported_constructs_raise_like_the_reference():
    """Constructs the reference cannot compile either raise its
    UnsupportedConstruct with its message (exprs.py:92-97)."""
    from paper_2506_22609_b200.errors import UnsupportedConstruct
    text = """(game "Dyn" (players 2) (equipment (board (square 5)) (pieces ("s" both)))
        (rules (play (repeat (P1 P2) (place "s" (destination (empty)))))
        (end (if (connected "s" ((edge top) (adjacent (occupied)))) (mover win)))))"""
    with pytest.raises(UnsupportedConstruct) as e:
        lowering.lower_game(syntax.parse_game(text))
    assert str(e.value) == "AdjacentMask is not static"
