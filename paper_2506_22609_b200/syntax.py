"""Reader for Ludax game text: s-expression tree first, AST second.

Design: a two-stage reader.  ``read_tree`` turns text into a tree of
``Form`` (parenthesised lists) and ``Tok`` (atoms, strings, keyword args),
then ``build_game`` interprets that tree form by form into ``nodes``.  The
accepted language is the reference grammar (reference:
pkg/src/boardlang/parser.py:17-1010; forms summarised in PAPER.md) -- the
same keywords, the same positional/keyword argument rules, and the same
node values -- so a program means here what it means to the reference.
"""

from __future__ import annotations

import re

from . import nodes as n
from .errors import ArityError, ParseError, UnknownKeywordError

_TOKEN = re.compile(r"""
    (?P<ws>\s+) | (?P<comment>//[^\n]*) | (?P<open>\() | (?P<close>\))
  | (?P<string>"[^"\n]*") | (?P<kwarg>[A-Za-z_][A-Za-z0-9_]*:)
  | (?P<variable>\?[a-z][a-z0-9]*) | (?P<atom>[A-Za-z0-9_=<>]+)
""", re.VERBOSE)
_INT = re.compile(r"(0|[1-9][0-9]*)\Z")


class Tok:
    __slots__ = ("kind", "text", "line", "col")

    def __init__(self, kind, text, line, col):
        self.kind, self.text, self.line, self.col = kind, text, line, col

    def __repr__(self):
        return f"{self.kind}:{self.text}"


class Form:
    """A parenthesised list; ``items`` holds Tok / Form children."""

    __slots__ = ("items", "line", "col")

    def __init__(self, items, line, col):
        self.items, self.line, self.col = items, line, col

    @property
    def head(self):
        if self.items and isinstance(self.items[0], Tok) and self.items[0].kind == "atom":
            return self.items[0].text
        return ""


def read_tree(text):
    """Text -> list of top-level Forms (comments and whitespace dropped)."""
    stack = [[]]
    opens = []
    pos, line, line_start = 0, 1, 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        col = pos - line_start + 1
        if m is None:
            raise ParseError(f"unexpected character {text[pos]!r}", line, col)
        kind, tt = m.lastgroup, m.group()
        if kind == "open":
            stack.append([])
            opens.append((line, col))
        elif kind == "close":
            if len(stack) == 1:
                raise ParseError("unbalanced ')'", line, col, {"("})
            items = stack.pop()
            ln, cl = opens.pop()
            stack[-1].append(Form(items, ln, cl))
        elif kind == "variable":
            raise UnknownKeywordError(f"variables ({tt}) are reserved and unsupported",
                                      line, col)
        elif kind not in ("ws", "comment"):
            stack[-1].append(Tok(kind, tt, line, col))
        nl = tt.count("\n")
        if nl:
            line += nl
            line_start = pos + tt.rfind("\n") + 1
        pos = m.end()
    if len(stack) != 1:
        ln, cl = opens[-1]
        raise ParseError("expected ')' before end of input", ln, cl, {")"})
    return stack[0]


# ---------------------------------------------------------------- helpers

def _loc(x):
    return (x.line, x.col)


def _fail(x, msg, cls=ParseError, expected=None):
    line, col = _loc(x) if x is not None else (None, None)
    raise cls(msg, line, col, expected)


class _Args:
    """Cursor over a form's items after its head keyword."""

    def __init__(self, form, skip=1, what=""):
        self.form = form
        self.items = form.items
        self.i = skip
        self.what = what or form.head

    def more(self):
        return self.i < len(self.items) and not self._is_kw(self.items[self.i])

    @staticmethod
    def _is_kw(x):
        return isinstance(x, Tok) and x.kind == "kwarg"

    def peek(self):
        return self.items[self.i] if self.i < len(self.items) else None

    def take(self):
        if self.i >= len(self.items):
            _fail(self.form, f"{self.what}: missing argument", ArityError)
        x = self.items[self.i]
        self.i += 1
        return x

    def form_(self):
        x = self.take()
        if not isinstance(x, Form):
            _fail(x, f"{self.what}: expected '(' got {x.text!r}", ParseError, {"("})
        return x

    def string(self, what):
        x = self.take()
        if not (isinstance(x, Tok) and x.kind == "string"):
            _fail(x, f"expected a quoted {what} name", ArityError)
        return x.text[1:-1]

    def integer(self, what, minimum=0):
        x = self.take()
        if not (isinstance(x, Tok) and x.kind == "atom" and _INT.match(x.text)):
            _fail(x, f"expected an integer for {what}", ArityError)
        v = int(x.text)
        if v < minimum:
            _fail(x, f"{what} must be >= {minimum}, got {v}", ArityError)
        return v

    def atom(self, choices, what, cls=UnknownKeywordError):
        x = self.take()
        if not (isinstance(x, Tok) and x.kind == "atom" and x.text in choices):
            got = x.text if isinstance(x, Tok) else "("
            _fail(x, f"expected {what}, got {got!r}", cls, set(choices))
        return x.text

    def kwargs(self, spec):
        out = {}
        while self.i < len(self.items):
            x = self.items[self.i]
            if not self._is_kw(x):
                _fail(x, f"unexpected {getattr(x, 'text', '(')!r} in {self.what}")
            name = x.text[:-1]
            if name not in spec:
                _fail(x, f"unknown keyword argument {x.text!r} in {self.what}",
                      UnknownKeywordError, {k + ":" for k in spec})
            if name in out:
                _fail(x, f"duplicate keyword argument {x.text!r} in {self.what}", ArityError)
            self.i += 1
            out[name] = spec[name](self)
        return out

    def done(self):
        if self.i < len(self.items):
            x = self.items[self.i]
            _fail(x, f"unexpected {getattr(x, 'text', '(')!r} in {self.what}")


_PLAYERS = {"P1": n.P1, "P2": n.P2}
_WHO = ("mover", "opponent")
_DIRS = set(n.TRUE_DIRECTIONS) | set(n.DIRECTION_GROUPS) | set(n.RELATIVE_DIRECTIONS)
_SHAPES = ("square", "rectangle", "hexagon", "hex_rectangle")
_FUNCTIONS = {"add", "connected", "count", "line", "multiply", "pattern", "score",
              "subtract"}
_PREDICATES = {"action_was", "can_move_again", "=", "exists", "full_board", ">=",
               "last_move_in", "<=", "mover_is", "no_legal_actions", "passed",
               "and", "or", "not"}
_MASKS = {"adjacent", "captured", "center", "column", "corners", "corner_custodial",
          "custodial", "edge", "empty", "hopped", "occupied", "prev_move", "promoted",
          "row", "region", "line", "and", "or", "not"}
_EFFECTS = {"capture", "extra_turn", "flip", "increment_score", "promote",
            "set_score", "if"}


def _who(a, players=False, both=False):
    x = a.take()
    if isinstance(x, Tok) and x.kind == "atom":
        if x.text in _WHO:
            return x.text
        if players and x.text in _PLAYERS:
            return _PLAYERS[x.text]
        if both and x.text == "both":
            return n.BOTH
    _fail(x, "expected a player reference", ArityError)


def _who_text(v):
    return {n.P1: "P1", n.P2: "P2"}.get(v, v) if isinstance(v, int) else v


def _bool(a):
    return a.atom(("true", "false"), "true/false", ArityError) == "true"


def _direction_value(a):
    x = a.take()
    if isinstance(x, Form):
        dirs = []
        for t in x.items:
            if not (isinstance(t, Tok) and t.text in _DIRS):
                _fail(t, "expected a direction", UnknownKeywordError, _DIRS)
            dirs.append(t.text)
        if not dirs:
            _fail(x, "direction list must not be empty", ArityError)
        return tuple(dirs)
    if not (isinstance(x, Tok) and x.text in _DIRS):
        _fail(x, "expected a direction", UnknownKeywordError, _DIRS)
    return (x.text,)


def _orientation(a):
    return a.atom(n.DIRECTION_GROUPS, "an orientation")


# ---------------------------------------------------------------- game

def parse_game(text):
    """Game text -> nodes.GameSpec (reference parser.py:1027 parse_game)."""
    top = read_tree(text)
    if not top:
        raise ParseError("expected '(' to open game", 1, 1, {"("})
    g = top[0]
    if not isinstance(g, Form) or g.head != "game":
        _fail(g, "expected (game ...)", ParseError, {"game"})
    if len(top) > 1:
        _fail(top[1], "unexpected form after game form")
    a = _Args(g)
    name = a.string("game")
    players = _players(a.form_())
    equipment = _equipment(a.form_())
    rules = a.form_()
    start, phases, end_rules = _rules(rules)
    rendering = None
    if a.peek() is not None:
        rf = a.form_()
        if rf.head != "rendering":
            _fail(rf, "expected (rendering ...)", ParseError, {"rendering"})
        rendering = _rendering(rf)
    a.done()
    return n.GameSpec(name=name, players=players, equipment=equipment, start=start,
                      phases=phases, end_rules=end_rules, rendering=rendering)


def _expect(form, head):
    if form.head != head:
        _fail(form, f"expected ({head} ...)", ParseError, {head})


def _players(f):
    _expect(f, "players")
    a = _Args(f)
    count = a.integer("player count", 1)
    forward = ()
    if a.peek() is not None:
        sf = a.form_()
        _expect(sf, "set_forward")
        b = _Args(sf)
        assigns = []
        for want in ("P1", "P2"):
            pf = b.form_()
            if pf.head != want:
                _fail(pf, f"expected {want}", ParseError, {want})
            c = _Args(pf)
            d = c.atom(("up", "down", "left", "right"), "up/down/left/right", ParseError)
            c.done()
            assigns.append((_PLAYERS[want], d))
        b.done()
        forward = tuple(assigns)
    a.done()
    return n.Players(count=count, forward=forward)


def _shape(f):
    kind = f.head
    if kind not in _SHAPES:
        _fail(f, "expected a board shape", UnknownKeywordError, set(_SHAPES))
    a = _Args(f)
    if kind == "square":
        shape = n.BoardShape("square", a.integer("board size", 1))
    elif kind == "hexagon":
        d = a.integer("hexagon diameter", 1)
        if d % 2 == 0:
            _fail(f, f"hexagon diameter must be odd, got {d}", ArityError)
        shape = n.BoardShape("hexagon", d)
    else:
        r = a.integer("row count", 1)
        c = a.integer("column count", 1)
        shape = n.BoardShape(kind, r, c)
    a.done()
    return shape


def _equipment(f):
    _expect(f, "equipment")
    a = _Args(f)
    bf = a.form_()
    _expect(bf, "board")
    b = _Args(bf)
    board = _shape(b.form_())
    b.done()
    pf = a.form_()
    _expect(pf, "pieces")
    pieces = []
    for item in pf.items[1:]:
        if not isinstance(item, Form):
            _fail(item, "expected a piece definition", ParseError, {"("})
        c = _Args(item, skip=0, what="piece definition")
        name = c.string("piece")
        owner = _who(c, players=True, both=True)
        if owner in _WHO:
            _fail(item, "piece owner must be P1, P2 or both", ArityError)
        c.done()
        pieces.append(n.PieceDef(name=name, owner=owner))
    if not pieces:
        _fail(pf, "pieces section must declare at least one piece", ArityError)
    regions = []
    if a.peek() is not None:
        rf = a.form_()
        _expect(rf, "regions")
        for item in rf.items[1:]:
            c = _Args(item, skip=0, what="region definition")
            name = c.string("region")
            cells, masks = _indices_or_masks(c.take())
            c.done()
            regions.append(n.RegionDef(name=name, cells=cells, masks=masks))
        if not regions:
            _fail(rf, "regions section must declare at least one region", ArityError)
    a.done()
    return n.Equipment(board=board, pieces=tuple(pieces), regions=tuple(regions))


def _indices_or_masks(x):
    if not isinstance(x, Form):
        _fail(x, "expected '('", ParseError, {"("})
    if x.items and isinstance(x.items[0], Tok) and _INT.match(x.items[0].text or ""):
        cells = []
        for t in x.items:
            if not (isinstance(t, Tok) and _INT.match(t.text)):
                _fail(t, "expected a cell index", ArityError)
            cells.append(int(t.text))
        return tuple(cells), ()
    return (), _multi_mask_arg(x)


def _multi_mask_arg(x):
    """multi-mask keyword | one super-mask | parenthesised super-mask list."""
    if not isinstance(x, Form):
        _fail(x, "expected a mask", ParseError, {"("})
    if x.head in ("edges", "edgesNoCorners", "corners") and len(x.items) == 1:
        return (n.MultiMask(x.head),)
    if not x.items:
        _fail(x, "mask list must not be empty", ArityError)
    if isinstance(x.items[0], Form):
        return tuple(mask(i) for i in x.items)
    return (mask(x),)


def _rules(f):
    _expect(f, "rules")
    a = _Args(f)
    start = ()
    x = a.form_()
    if x.head == "start":
        start = _start(x)
        x = a.form_()
    _expect(x, "play")
    phases = tuple(_phase(p) for p in x.items[1:])
    if not phases:
        _fail(x, "play section must contain at least one phase", ArityError)
    ef = a.form_()
    _expect(ef, "end")
    rules = []
    for r in ef.items[1:]:
        if not isinstance(r, Form) or r.head != "if":
            _fail(r, "expected (if ...)", ParseError, {"if"})
        b = _Args(r)
        cond = predicate(b.take())
        res = _end_result(b.form_())
        b.done()
        rules.append(n.EndRule(condition=cond, result=res))
    if not rules:
        _fail(ef, "end section must contain at least one rule", ArityError)
    a.done()
    return start, phases, tuple(rules)


def _start(f):
    out = []
    for item in f.items[1:]:
        if not isinstance(item, Form) or item.head != "place":
            _fail(item, "expected (place ...)", ParseError, {"place"})
        a = _Args(item)
        piece = a.string("piece")
        player = _PLAYERS[a.atom(("P1", "P2"), "P1 or P2", ArityError)]
        cells, masks = _indices_or_masks(a.take())
        a.done()
        out.append(n.StartPlace(piece=piece, player=player, cells=cells, masks=masks))
    if not out:
        _fail(f, "start section must contain at least one placement", ArityError)
    return tuple(out)


def _phase(f):
    if not isinstance(f, Form) or f.head not in ("repeat", "once_through"):
        _fail(f, "expected repeat or once_through", UnknownKeywordError,
              {"repeat", "once_through"})
    a = _Args(f)
    of = a.form_()
    order = []
    for t in of.items:
        if not (isinstance(t, Tok) and t.text in _PLAYERS):
            _fail(t, "expected P1 or P2", ArityError)
        order.append(_PLAYERS[t.text])
    if not order:
        _fail(of, "mover order must name at least one player", ArityError)
    mf = a.form_()
    if mf.head == "place":
        mech = _place(mf)
    elif mf.head == "move":
        mech = _move(mf)
    else:
        _fail(mf, "expected place or move", UnknownKeywordError, {"place", "move"})
    force_pass = False
    if a.peek() is not None:
        fp = a.form_()
        _expect(fp, "force_pass")
        force_pass = True
    a.done()
    return n.Phase(kind=f.head, order=tuple(order), mechanic=mech, force_pass=force_pass)


def _place(f):
    a = _Args(f)
    piece = a.string("piece")
    owner = n.MOVER
    x = a.peek()
    if isinstance(x, Tok) and x.text in _WHO:
        owner = a.take().text
    df = a.form_()
    _expect(df, "destination")
    d = _Args(df)
    dest = mask(d.take())
    d.done()
    result, effects = None, ()
    while a.peek() is not None:
        x = a.form_()
        if x.head == "result" and result is None and not effects:
            r = _Args(x)
            result = predicate(r.take())
            r.done()
        elif x.head == "effects" and not effects:
            effects = _effects(x)
        else:
            _fail(x, f"unexpected ({x.head} ...) in place", ParseError)
    return n.PlaceMechanic(piece=piece, owner=owner, destination=dest, result=result,
                           effects=effects)


def _move(f):
    a = _Args(f)
    first = a.form_()
    if first.head == "or":
        moves = tuple(_move_type(m) for m in first.items[1:])
        if not moves:
            _fail(first, "move (or ...) needs at least one move type", ArityError)
    else:
        moves = (_move_type(first),)
    effects = ()
    if a.peek() is not None:
        ef = a.form_()
        _expect(ef, "effects")
        effects = _effects(ef)
    a.done()
    return n.MoveMechanic(moves=moves, effects=effects)


def _move_type(f):
    if not isinstance(f, Form) or f.head not in n.MOVE_KINDS:
        _fail(f, "expected hop, slide or step", UnknownKeywordError, set(n.MOVE_KINDS))
    a = _Args(f)
    piece = a.string("piece")
    if f.head == "hop":
        kw = a.kwargs({"direction": _direction_value,
                       "piece": lambda b: b.string("piece"),
                       "hop_over": lambda b: _who(b, players=True),
                       "capture": _bool,
                       "priority": lambda b: b.integer("priority")})
        return n.HopMove(piece=piece, directions=kw.get("direction", ()),
                         over_piece=kw.get("piece", ""),
                         hop_over=_who_text(kw.get("hop_over", "")),
                         capture=kw.get("capture", False), priority=kw.get("priority", 0))
    if f.head == "slide":
        kw = a.kwargs({"direction": _direction_value,
                       "distance": lambda b: b.integer("distance", 1),
                       "priority": lambda b: b.integer("priority")})
        return n.SlideMove(piece=piece, directions=kw.get("direction", ()),
                           distance=kw.get("distance", 0), priority=kw.get("priority", 0))
    kw = a.kwargs({"direction": _direction_value,
                   "priority": lambda b: b.integer("priority")})
    return n.StepMove(piece=piece, directions=kw.get("direction", ()),
                      priority=kw.get("priority", 0))


def _effects(f):
    out = tuple(_effect(e, True) for e in f.items[1:])
    if not out:
        _fail(f, "effects section must contain at least one effect", ArityError)
    return out


def _effect(f, allow_if):
    if not isinstance(f, Form) or f.head not in _EFFECTS or (f.head == "if" and not allow_if):
        _fail(f, "expected an effect", UnknownKeywordError, _EFFECTS)
    a = _Args(f)
    h = f.head
    if h == "if":
        cond = predicate(a.take())
        then = _effect(a.form_(), False)
        other = None
        x = a.peek()
        if isinstance(x, Tok) and x.text == "else":
            a.take()
            other = _effect(a.form_(), False)
        a.done()
        return n.ConditionalEffect(condition=cond, then_effect=then, else_effect=other)
    if h == "capture":
        m = mask(a.take())
        kw = a.kwargs({"mover": lambda b: _who(b, both=True), "increment_score": _bool})
        return n.CaptureEffect(mask=m, mover=kw.get("mover", n.MOVER),
                               increment_score=kw.get("increment_score", False))
    if h == "extra_turn":
        who = _who(a)
        kw = a.kwargs({"same_piece": _bool})
        return n.ExtraTurnEffect(who=who, same_piece=kw.get("same_piece", False))
    if h == "flip":
        m = mask(a.take())
        kw = a.kwargs({"mover": lambda b: _who(b, both=True)})
        return n.FlipEffect(mask=m, mover=kw.get("mover", n.MOVER))
    if h == "promote":
        fp = a.string("piece")
        tp = a.string("piece")
        m = mask(a.take())
        kw = a.kwargs({"mover": lambda b: _who(b, both=True)})
        return n.PromoteEffect(from_piece=fp, to_piece=tp, mask=m,
                               mover=kw.get("mover", n.MOVER))
    who = _who(a)
    fn = function(a.take())
    a.done()
    if h == "increment_score":
        return n.IncrementScoreEffect(who=who, fn=fn)
    return n.SetScoreEffect(who=who, fn=fn)


def _end_result(f):
    items = f.items
    if len(items) == 1 and isinstance(items[0], Tok) and items[0].text in ("draw", "by_score"):
        return n.EndResult(kind=items[0].text)
    if (len(items) == 2 and all(isinstance(t, Tok) for t in items)
            and items[0].text in ("mover", "opponent", "both")
            and items[1].text in ("win", "lose")):
        return n.EndResult(kind=items[1].text, who=items[0].text)
    _fail(f, "expected an end result", UnknownKeywordError,
          {"mover", "opponent", "both", "draw", "by_score"})


def _rendering(f):
    colors, shapes = [], []
    for item in f.items[1:]:
        if not isinstance(item, Form) or item.head not in ("color", "shape"):
            _fail(item, "expected color or shape", UnknownKeywordError, {"color", "shape"})
        a = _Args(item)
        if item.head == "color":
            p = _PLAYERS[a.atom(("P1", "P2"), "P1 or P2", ArityError)]
            colors.append((p, a.atom(("white", "black"), "white or black")))
        else:
            pc = a.string("piece")
            shapes.append((pc, a.atom(n.PIECE_SHAPES, "a piece shape")))
        a.done()
    if not colors and not shapes:
        _fail(f, "rendering section must contain at least one detail", ArityError)
    return n.Rendering(colors=tuple(colors), shapes=tuple(shapes))


# ---------------------------------------------------------------- expressions

def mask(x):
    """Super-mask form -> mask node (reference parser.py:702-811)."""
    if not isinstance(x, Form):
        _fail(x, "expected a mask", ParseError, {"("})
    h = x.head
    if h not in _MASKS:
        _fail(x, f"unknown mask {h!r}", UnknownKeywordError, _MASKS)
    if h in ("and", "or", "not"):
        items = tuple(mask(i) for i in x.items[1:])
        if not items:
            _fail(x, f"({h} ...) mask needs at least one operand", ArityError)
        if h == "not":
            if len(items) != 1:
                _fail(x, "(not ...) mask takes exactly one operand", ArityError)
            return n.MaskNot(items[0])
        return n.MaskAnd(items) if h == "and" else n.MaskOr(items)
    if h == "line":
        return _line(x)
    a = _Args(x)
    if h == "adjacent":
        inner = mask(a.take())
        kw = a.kwargs({"direction": _direction_value})
        return n.AdjacentMask(inner=inner, directions=kw.get("direction", ()))
    if h == "custodial":
        piece = a.string("piece")
        t = a.take()
        if isinstance(t, Tok) and t.text == "any":
            length = "any"
        elif isinstance(t, Tok) and _INT.match(t.text) and int(t.text) >= 1:
            length = int(t.text)
        else:
            _fail(t, "custodial length must be a positive integer or any", ArityError)
        kw = a.kwargs({"mover": lambda b: _who(b, both=True), "orientation": _orientation})
        return n.CustodialMask(piece=piece, length=length, mover=kw.get("mover", n.MOVER),
                               orientation=kw.get("orientation", "any"))
    if h == "corner_custodial":
        piece = a.string("piece")
        kw = a.kwargs({"mover": lambda b: _who(b, both=True)})
        return n.CornerCustodialMask(piece=piece, mover=kw.get("mover", n.MOVER))
    if h == "edge":
        which = a.atom(set(n.EDGE_NAMES) | {"forward", "backward"}, "an edge name")
        node = n.EdgeMask(which=which)
    elif h == "occupied":
        who = ""
        t = a.peek()
        if isinstance(t, Tok) and t.text in _WHO:
            who = a.take().text
        node = n.OccupiedMask(who=who)
    elif h in ("column", "row"):
        idx = a.integer(f"{h} index")
        node = n.ColumnMask(index=idx) if h == "column" else n.RowMask(index=idx)
    elif h == "region":
        node = n.RegionMask(region=a.string("region"))
    elif h == "prev_move":
        node = n.PrevMoveMask(who=_who(a))
    else:
        node = {"captured": n.CapturedMask, "center": n.CenterMask,
                "corners": n.CornersMask, "empty": n.EmptyMask,
                "hopped": n.HoppedMask, "promoted": n.PromotedMask}[h]()
    a.done()
    return node


def _line(x):
    a = _Args(x)
    piece = a.string("piece")
    length = a.integer("line length", 1)
    kw = a.kwargs({"orientation": _orientation, "exact": _bool,
                   "player": lambda b: _who(b, players=True),
                   "exclude": lambda b: _multi_mask_arg(b.take())})
    ex = kw.get("exclude")
    if ex is not None and len(ex) == 1 and isinstance(ex[0], n.MultiMask):
        ex = ex[0]
    return n.LineFn(piece=piece, length=length, orientation=kw.get("orientation", "any"),
                    exact=kw.get("exact", False),
                    player=_who_text(kw.get("player", n.MOVER)), exclude=ex)


def _pattern(x):
    a = _Args(x)
    piece = a.string("piece")
    arg = a.form_()
    width, offsets, shape = 0, (), None
    if arg.head in _SHAPES:
        shape = _shape(arg)
    else:
        b = _Args(arg, skip=0, what="pattern argument")
        width = b.integer("pattern width", 1)
        of = b.form_()
        offsets = tuple(int(t.text) for t in of.items
                        if isinstance(t, Tok) and _INT.match(t.text))
        if not offsets or len(offsets) != len(of.items):
            _fail(of, "pattern offsets must be a non-empty integer list", ArityError)
        b.done()
    kw = a.kwargs({"rotate": _bool, "player": lambda b: _who(b, players=True),
                   "exclude": lambda b: _multi_mask_arg(b.take())})
    ex = kw.get("exclude")
    if ex is not None and len(ex) == 1 and isinstance(ex[0], n.MultiMask):
        ex = ex[0]
    return n.PatternFn(piece=piece, width=width, offsets=offsets, shape=shape,
                       rotate=kw.get("rotate", False),
                       player=_who_text(kw.get("player", n.MOVER)), exclude=ex)


def function(x):
    """Function form -> function node (reference parser.py:815-905)."""
    if isinstance(x, Tok) and x.kind == "atom" and _INT.match(x.text):
        v = int(x.text)
        if v < 1:
            _fail(x, "constant must be >= 1", ArityError)
        return n.ConstantFn(value=v)
    if not isinstance(x, Form):
        _fail(x, "expected a function", ParseError, {"("})
    h = x.head
    if h == "line":
        return _line(x)
    if h == "pattern":
        return _pattern(x)
    if h not in _FUNCTIONS:
        _fail(x, f"unknown function {h!r}", UnknownKeywordError, _FUNCTIONS)
    a = _Args(x)
    if h in ("add", "multiply"):
        items = tuple(function(i) for i in x.items[1:])
        if not items:
            _fail(x, f"({h} ...) needs at least one operand", ArityError)
        return n.AddFn(items) if h == "add" else n.MultiplyFn(items)
    if h == "connected":
        piece = a.string("piece")
        masks = _multi_mask_arg(a.take())
        kw = a.kwargs({"mover": lambda b: _who(b, both=True),
                       "direction": _direction_value})
        if len(masks) == 1 and isinstance(masks[0], n.MultiMask):
            masks = masks[0]
        return n.ConnectedFn(piece=piece, masks=masks, mover=kw.get("mover", n.MOVER),
                             directions=kw.get("direction", ()))
    if h == "count":
        node = n.CountFn(mask=mask(a.take()))
    elif h == "score":
        node = n.ScoreFn(who=_who(a))
    else:
        node = n.SubtractFn(a=function(a.take()), b=function(a.take()))
    a.done()
    return node


def predicate(x):
    """Super-predicate -> predicate node (reference parser.py:950-1010)."""
    if isinstance(x, Tok) and x.kind == "atom" and _INT.match(x.text):
        return n.FunctionPred(fn=function(x))
    if not isinstance(x, Form):
        _fail(x, "expected a predicate", ParseError, {"("})
    h = x.head
    if h in ("and", "or", "not"):
        items = tuple(predicate(i) for i in x.items[1:])
        if not items:
            _fail(x, f"({h} ...) predicate needs at least one operand", ArityError)
        if h == "not":
            if len(items) != 1:
                _fail(x, "(not ...) predicate takes exactly one operand", ArityError)
            return n.PredNot(items[0])
        return n.PredAnd(items) if h == "and" else n.PredOr(items)
    if h in _FUNCTIONS and h not in _PREDICATES:
        return n.FunctionPred(fn=function(x))
    if h not in _PREDICATES:
        _fail(x, f"unknown predicate {h!r}", UnknownKeywordError, _PREDICATES | _FUNCTIONS)
    a = _Args(x)
    if h in ("action_was", "can_move_again"):
        who = _who(a) if h == "action_was" else None
        kind = a.atom(n.MOVE_KINDS, "hop, slide or step")
        node = n.ActionWasPred(who=who, kind=kind) if who else n.CanMoveAgainPred(kind=kind)
    elif h == "=":
        items = []
        while a.more():
            items.append(function(a.take()))
        if len(items) < 2:
            _fail(x, "(= ...) needs at least two functions", ArityError)
        node = n.EqualsPred(items=tuple(items))
    elif h in (">=", "<="):
        fa, fb = function(a.take()), function(a.take())
        node = n.GreaterEqPred(a=fa, b=fb) if h == ">=" else n.LessEqPred(a=fa, b=fb)
    elif h in ("exists", "last_move_in"):
        m = mask(a.take())
        node = n.ExistsPred(mask=m) if h == "exists" else n.LastMoveInPred(mask=m)
    elif h == "mover_is":
        node = n.MoverIsPred(player=_PLAYERS[a.atom(("P1", "P2"), "P1 or P2", ArityError)])
    elif h == "passed":
        node = n.PassedPred(who=_who(a, both=True))
    else:
        node = {"full_board": n.FullBoardPred,
                "no_legal_actions": n.NoLegalActionsPred}[h]()
    a.done()
    return node
