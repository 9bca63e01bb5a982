"""Board geometry on the host: cell numbering, neighbours, edges, lines.

This is host-side only: the lowering turns these tables into per-direction
bit-shift amounts plus validity masks (``lowering.py``), and proves the two
agree cell by cell.  Conventions follow the reference topology (reference:
pkg/src/boardlang/topology.py:1-460): cells are numbered row-major from the
top-left; square/rectangle boards use (row, col) with eight directions;
hex_rectangle boards use (row, col) with the six axial neighbours
(0,+-1), (+-1,0), (-1,+1), (+1,-1); hexagon boards use axial (q, r).
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidShapeParam, MissingForwardAssignment

SQUARE_DIRS = ("up", "down", "left", "right", "up_left", "up_right",
               "down_left", "down_right")
HEXAGON_DIRS = ("left", "right", "up_left", "up_right", "down_left", "down_right")
HEX_RECT_DIRS = ("left", "right", "up", "down", "up_right", "down_left")

OPPOSITE = {"up": "down", "down": "up", "left": "right", "right": "left",
            "up_left": "down_right", "down_right": "up_left",
            "up_right": "down_left", "down_left": "up_right"}

# (delta_a, delta_b) per family; a/b = row/col on grids, q/r on hexagons
_DELTAS = {
    "grid": {"up": (-1, 0), "down": (1, 0), "left": (0, -1), "right": (0, 1),
             "up_left": (-1, -1), "up_right": (-1, 1),
             "down_left": (1, -1), "down_right": (1, 1)},
    "hex_rectangle": {"left": (0, -1), "right": (0, 1), "up": (-1, 0), "down": (1, 0),
                      "up_right": (-1, 1), "down_left": (1, -1)},
    "hexagon": {"left": (-1, 0), "right": (1, 0), "up_left": (0, -1),
                "up_right": (1, -1), "down_left": (-1, 1), "down_right": (0, 1)},
}

_GROUPS = {
    "grid": {"vertical": ("up", "down"), "horizontal": ("left", "right"),
             "orthogonal": ("up", "down", "left", "right"),
             "diagonal": ("up_left", "up_right", "down_left", "down_right"),
             "back_diagonal": ("up_left", "down_right"),
             "forward_diagonal": ("up_right", "down_left"), "any": SQUARE_DIRS},
    "hexagon": {"horizontal": ("left", "right"),
                "diagonal": ("up_left", "up_right", "down_left", "down_right"),
                "back_diagonal": ("up_left", "down_right"),
                "forward_diagonal": ("up_right", "down_left"), "any": HEXAGON_DIRS},
    "hex_rectangle": {"vertical": ("up", "down"), "horizontal": ("left", "right"),
                      "orthogonal": ("up", "down", "left", "right"),
                      "diagonal": ("up_right", "down_left"),
                      "forward_diagonal": ("up_right", "down_left"),
                      "any": HEX_RECT_DIRS},
}

# line / custodial orientation keyword -> one walk direction per axis
_ORIENT = {
    "grid": {"horizontal": ("right",), "vertical": ("down",),
             "forward_diagonal": ("down_left",), "back_diagonal": ("down_right",),
             "diagonal": ("down_left", "down_right"), "orthogonal": ("right", "down"),
             "any": ("right", "down", "down_right", "down_left")},
    "hexagon": {"horizontal": ("right",), "forward_diagonal": ("down_left",),
                "back_diagonal": ("down_right",),
                "diagonal": ("down_left", "down_right"),
                "any": ("right", "down_left", "down_right")},
    "hex_rectangle": {"horizontal": ("right",), "vertical": ("down",),
                      "forward_diagonal": ("down_left",), "diagonal": ("down_left",),
                      "orthogonal": ("right", "down"),
                      "any": ("right", "down", "down_left")},
}

_RELATIVE = {
    "up": {"forward": "up", "backward": "down", "forward_left": "up_left",
           "forward_right": "up_right", "backward_left": "down_left",
           "backward_right": "down_right"},
    "down": {"forward": "down", "backward": "up", "forward_left": "down_right",
             "forward_right": "down_left", "backward_left": "up_right",
             "backward_right": "up_left"},
    "left": {"forward": "left", "backward": "right", "forward_left": "down_left",
             "forward_right": "up_left", "backward_left": "down_right",
             "backward_right": "up_right"},
    "right": {"forward": "right", "backward": "left", "forward_left": "up_right",
              "forward_right": "down_right", "backward_left": "up_left",
              "backward_right": "down_left"},
}


class Board:
    """Immutable geometry of one board shape."""

    def __init__(self, shape):
        kind = shape.kind
        if kind in ("square", "rectangle", "hex_rectangle"):
            rows, cols = shape.rows, shape.cols
            if rows < 1 or cols < 1:
                raise InvalidShapeParam(f"board dimensions must be positive: {rows}x{cols}")
            coords = [(r, c) for r in range(rows) for c in range(cols)]
            family = "hex_rectangle" if kind == "hex_rectangle" else "grid"
        elif kind == "hexagon":
            d = shape.rows
            if d < 1 or d % 2 == 0:
                raise InvalidShapeParam(f"hexagon diameter must be odd and positive: {d}")
            rad = (d - 1) // 2
            coords = [(q, r) for r in range(-rad, rad + 1)
                      for q in range(max(-rad, -rad - r), min(rad, rad - r) + 1)]
            rows = cols = d
            family = "hexagon"
            self.radius = rad
        else:
            raise InvalidShapeParam(f"unknown board shape {kind!r}")
        self.kind, self.family = kind, family
        self.rows, self.cols = rows, cols
        self.coords = coords
        self.num_cells = C = len(coords)
        self.sentinel = C
        self._index = {c: i for i, c in enumerate(coords)}
        self.directions = {"grid": SQUARE_DIRS, "hex_rectangle": HEX_RECT_DIRS,
                           "hexagon": HEXAGON_DIRS}[family]
        if family == "hexagon":
            self.row_of = np.array([r + self.radius for _, r in coords], dtype=np.int16)
            first = {}
            for i, r in enumerate(self.row_of.tolist()):
                first.setdefault(r, i)
            self.col_of = np.array([i - first[r] for i, r in enumerate(self.row_of.tolist())],
                                   dtype=np.int16)
        else:
            self.row_of = np.array([a for a, _ in coords], dtype=np.int16)
            self.col_of = np.array([b for _, b in coords], dtype=np.int16)

        self.neighbors = {}
        for dname in self.directions:
            da, db = _DELTAS[family][dname]
            t = np.full(C + 1, C, dtype=np.int16)
            for i, (a, b) in enumerate(coords):
                j = self._index.get((a + da, b + db))
                if j is not None:
                    t[i] = j
            self.neighbors[dname] = t
        self._edges()
        self._center()

    # -- static masks --

    def mask_of(self, cells):
        m = np.zeros(self.num_cells, dtype=bool)
        m[list(cells)] = True
        return m

    def _edges(self):
        row, col = self.row_of, self.col_of
        e = {}
        if self.family == "hexagon":
            d, rad = self.rows, self.radius
            first = col == 0
            last = np.zeros(self.num_cells, dtype=bool)
            for r in range(d):
                last[np.nonzero(row == r)[0][-1]] = True
            top, bot = row <= rad, row >= rad
            e = {"top": row == 0, "bottom": row == d - 1,
                 "top_left": first & top, "top_right": last & top,
                 "bottom_left": first & bot, "bottom_right": last & bot}
            corners = []
            for r in (0, rad, d - 1):
                idx = np.nonzero(row == r)[0]
                corners += [int(idx[0]), int(idx[-1])]
            self.corner_cells = tuple(sorted(corners))
            self.edge_order = ("top", "top_right", "bottom_right", "bottom",
                               "bottom_left", "top_left")
        else:
            e = {"top": row == 0, "bottom": row == self.rows - 1,
                 "left": col == 0, "right": col == self.cols - 1}
            for nm, (a, b) in (("top_left", ("top", "left")), ("top_right", ("top", "right")),
                               ("bottom_left", ("bottom", "left")),
                               ("bottom_right", ("bottom", "right"))):
                e[nm] = e[a] & e[b]
            self.corner_cells = tuple(int(np.nonzero(e[nm])[0][0]) for nm in
                                      ("top_left", "top_right", "bottom_left", "bottom_right"))
            self.edge_order = ("top", "bottom", "left", "right")
        self.edge_masks = e
        self.corners_mask = self.mask_of(self.corner_cells)

    def _center(self):
        if self.family == "hexagon":
            self.center_mask = self.mask_of([self._index[(0, 0)]])
            return

        def mid(k):
            return (k // 2,) if k % 2 else (k // 2 - 1, k // 2)
        self.center_mask = self.mask_of(
            [self._index[(r, c)] for r in mid(self.rows) for c in mid(self.cols)])

    def multi_mask(self, kind):
        if kind == "edges":
            return [self.edge_masks[k] for k in self.edge_order]
        if kind == "corners":
            return [self.mask_of([c]) for c in self.corner_cells]
        if kind == "edgesNoCorners":
            return [self.edge_masks[k] & ~self.corners_mask for k in self.edge_order]
        raise KeyError(kind)

    # -- direction vocabulary --

    def expand(self, word):
        if word in self.directions:
            return (word,)
        groups = _GROUPS[self.family]
        if word in groups:
            return groups[word]
        raise KeyError(f"direction {word!r} is not available on a {self.kind} board")

    def orientation_dirs(self, word):
        if word in self.directions:
            return (word,)
        orients = _ORIENT[self.family]
        if word in orients:
            return orients[word]
        raise KeyError(f"orientation {word!r} is not available on a {self.kind} board")

    def coord_of(self, cell):
        return self.coords[cell]

    def cell_at(self, coord):
        return self._index.get(tuple(coord))

    def delta(self, direction):
        return _DELTAS[self.family][direction]

    def ray_length(self, direction):
        """Longest walk (in cells, excluding the start) along a direction."""
        nt = self.neighbors[direction]
        best = 0
        for c in range(self.num_cells):
            k, x = 0, c
            while nt[x] != self.sentinel:
                x = int(nt[x])
                k += 1
            best = max(best, k)
        return best

    def line_windows(self, length, orientation):
        """All windows (start, walk-direction) of ``length`` cells."""
        out = []
        for d in self.orientation_dirs(orientation):
            nt = self.neighbors[d]
            for s in range(self.num_cells):
                cells = [s]
                while len(cells) < length and nt[cells[-1]] != self.sentinel:
                    cells.append(int(nt[cells[-1]]))
                if len(cells) == length:
                    out.append((d, tuple(cells)))
        return out


def resolve_direction(tokens, player, forward_map, board):
    """Direction tokens -> ordered true directions (reference topology.py:433-460)."""
    if not tokens:
        tokens = ("any",)
    out = []
    for word in tokens:
        if word in _RELATIVE["up"]:
            facing = forward_map.get(player)
            if facing is None:
                raise MissingForwardAssignment(
                    f"direction {word!r} needs (set_forward ...) for player {player + 1}")
            word = _RELATIVE[facing][word]
            if word not in board.directions:
                raise KeyError(f"direction {word!r} is not available on a {board.kind} board")
            out.append(word)
        else:
            out.extend(board.expand(word))
    return tuple(d for d in board.directions if d in out)


def direction_pairs(tokens, forward_map, board):
    """Per-slot (P1 direction, P2 direction) pairs (reference mechanics.py:25-41)."""
    if not tokens:
        tokens = ("any",)
    pairs = []
    for word in tokens:
        d1 = resolve_direction((word,), 0, forward_map, board)
        d2 = resolve_direction((word,), 1, forward_map, board)
        if len(d1) == len(d2):
            pairs.extend(zip(d1, d2))
        else:
            pairs.extend((d, d) for d in d1)
    out = []
    for p in pairs:
        if p not in out:
            out.append(p)
    return tuple(out)
