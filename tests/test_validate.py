"""Semantic validation identical to the reference's (validate.py): the same
report, path for path and message for message, on 600 programs from the
reference's generator, most of them invalid (tests/golden/validate.json)."""
import json
import os

import pytest

from conftest import GOLDEN, game_text
from paper_2506_22609_b200 import syntax
from paper_2506_22609_b200.errors import ValidationFailure
from paper_2506_22609_b200.validate import validate

with open(os.path.join(GOLDEN, "validate.json")) as f:
    CASES = json.load(f)


def report_of(text):
    try:
        return str(validate(syntax.parse_game(text)))
    except Exception as exc:
        return f"EXC {type(exc).__name__}: {exc}"


def test_validation_reports_match_reference():
    mism = [(c["sampler"], c["index"]) for c in CASES if report_of(c["text"]) != c["report"]]
    assert not mism, mism[:10]
    assert sum(c["report"] == "valid" for c in CASES) >= 100


def test_load_game_raises_validation_failure():
    import paper_2506_22609_b200 as lx
    bad = next(c for c in CASES if c["report"] != "valid" and not c["report"].startswith("EXC"))
    with pytest.raises(ValidationFailure) as e:
        lx.load_game(bad["text"])
    assert str(e.value) == bad["report"]


@pytest.mark.parametrize("name", ["tic_tac_toe", "english_draughts", "yavalath", "gridworld"])
def test_corpus_games_are_valid(name):
    assert validate(syntax.parse_game(game_text(name))).ok
