"""Lowering: parsed game AST -> one CUDA translation unit per game.

The reference compiles each AST node into a numpy closure over (B, C)
arrays (reference: pkg/src/boardlang/compiler.py:197-650, exprs.py,
effects.py, mechanics.py:415-515).  Here every node becomes a fragment of a
``struct Game`` whose device functions operate on one env's bitboards held
in registers; ``csrc/device/lx_kernels.cuh`` then instantiates the kernels
(init, legal, sample, step, fused rollout, export/import) around it and the
native runtime compiles the unit with NVRTC for sm_100a.

Supported subset (the five config games): placement
mechanics on square / rectangle / hex_rectangle boards with one piece type;
masks empty/occupied/edge/center/corners/row/column/region/adjacent/
and/or/not and custodial (as placement result and as flip/capture effect);
functions count/score/constant/line/connected/add/multiply/subtract;
predicates and/or/not/exists/full_board/mover_is/>=/<=/=/passed/line;
effects flip/capture/set_score/increment_score/if; phases repeat /
once_through / force_pass; results win/lose/draw/by_score.  Anything else
raises CompileError("lower", ...) -- there is no CPU fallback.
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass, field

import numpy as np

from . import nodes as n
from .errors import CompileError, UnsupportedConstruct
from .geometry import OPPOSITE, Board, direction_pairs, resolve_direction
from .lowering_moves import KIND_IDS, MoveLoweringMixin

ANCHOR_COST_THRESHOLD = 128          # reference compiler.py:28


def _fail(msg):
    raise CompileError("lower", msg)


@dataclass
class Lowered:
    name: str
    source: str
    info: dict = field(default_factory=dict)

    @property
    def key(self):
        return hashlib.sha256(self.source.encode()).hexdigest()[:24]


class _Emitter:
    """Collects constants and helper functions while expressions are built."""

    def __init__(self, board, W, bit_of):
        self.board, self.W = board, W
        self.bit_of = bit_of      # cell id -> bit position
        self.consts = {}          # words tuple -> name
        self.helpers = {}         # name -> code
        self.counter = 0

    def const(self, mask):
        """Constant bitboard from a cell-indexed bool mask."""
        bits = np.zeros(self.W * 32, dtype=bool)
        bits[self.bit_of[np.nonzero(np.asarray(mask))[0]]] = True
        words = _words(bits, self.W)
        if words not in self.consts:
            self.consts[words] = f"K{len(self.consts)}"
        return f"{self.consts[words]}()"

    def fresh(self, base="t"):
        self.counter += 1
        return f"{base}{self.counter}"

    def helper(self, name, code):
        self.helpers.setdefault(name, code)
        return name

    def const_defs(self):
        out = []
        for words, name in self.consts.items():
            lit = ", ".join(f"0x{w:08x}u" for w in words)
            out.append(f"    static __device__ __forceinline__ BBW {name}() {{ return BBW{{{{{lit}}}}}; }}")
        return "\n".join(out)


def _words(mask, W):
    m = np.zeros(W * 32, dtype=bool)
    m[:len(mask)] = mask
    return tuple(int(x) for x in np.packbits(m.reshape(W, 32)[:, ::-1], axis=1)
                 .view(">u4").reshape(W))


class GameLowering(MoveLoweringMixin):
    """Walks one validated GameSpec and produces its Lowered unit."""

    def __init__(self, spec):
        self.spec = spec
        self.board = Board(spec.equipment.board)
        B = self.board
        self.C = B.num_cells
        # Bit layout.  Row-major boards: bit = cell.  Hexagon boards: rows of
        # different lengths are embedded in a d x d axial grid (row r, column
        # q + radius), which makes every direction a constant shift; bit order
        # stays monotone in cell order, so "r-th set bit" is still the r-th
        # legal cell (reference mechanics.py:488-492).
        if B.family == "hexagon":
            d, rad = B.rows, B.radius
            self.emb_rows = self.emb_cols = d
            self.bit_of = np.array([(r + rad) * d + (q + rad) for q, r in B.coords])
        else:
            self.emb_rows, self.emb_cols = B.rows, B.cols
            self.bit_of = np.arange(self.C)
        self.NB = self.emb_rows * self.emb_cols
        self.ident = bool((self.bit_of == np.arange(self.C)).all())
        self.W = (self.NB + 31) // 32
        self.em = _Emitter(B, self.W, self.bit_of)
        self.rm_used = False            # a probe was lowered onto the row mirror
        self.piece_ids = {p.name: i for i, p in enumerate(spec.equipment.pieces)}
        self._setup_piece_types()
        self.anchored_ctx = False          # effects compile with the anchored context
        self.forward = dict(spec.players.forward)
        self.regions = {}
        for r in spec.equipment.regions:
            self.regions[r.name] = (B.mask_of(r.cells) if r.cells
                                    else self._static_union(r.masks))
        self.valid = np.ones(self.C, dtype=bool)
        self._shift = {}
        for d in B.directions:
            self._shift[d] = self._check_shift(d)
        self.conn_plans = []
        self._scan()

    # ------------------------------------------------------------ geometry

    def _check_shift(self, d):
        """Prove bit(nbr_d(x)) == bit(x) + S for every x with a d-neighbour."""
        nt = self.board.neighbors[d]
        bo = self.bit_of
        deltas = {int(bo[nt[x]]) - int(bo[x]) for x in range(self.C) if nt[x] != self.C}
        if len(deltas) > 1:
            _fail(f"direction {d} is not a constant cell shift on this board")
        return deltas.pop() if deltas else 0

    def _walk_ok(self, d, k):
        nt = self.board.neighbors[d]
        x = np.arange(self.C)
        for _ in range(k):
            x = nt[x]
        return x != self.C

    def walk(self, d, k, expr):
        """Expression: bit x = expr bit (x + k*S_d), masked to valid walks."""
        S = self._shift[d] * k
        name = f"walk_{d}_{k}"
        mask = self.em.const(self._walk_ok(d, k))
        self.em.helper(name, f"    static __device__ __forceinline__ BBW {name}(const BBW& x) "
                             f"{{ return lx::gather<W, {S}>(x) & {mask}; }}\n"
                             f"#if defined(__CUDA_ARCH__)\n"
                             f"    static __device__ __forceinline__ lx::LW<W> {name}(const lx::LW<W>& x) "
                             f"{{ return lx::gather<W, {S}>(x) & {mask}; }}\n"
                             f"#endif")
        return f"{name}({expr})"

    def nb(self, d, expr):
        """neighbour gather: bit x = expr bit at nbr_d(x) (0 off-board)."""
        return self.walk(d, 1, expr)

    # ------------------------------------------------------------ scan / layout

    def _scan(self):
        """StateLayout + codec facts (reference compiler.py:98-152, 200-221)."""
        spec = self.spec
        allnodes = list(n.walk(spec))
        types = {type(x) for x in allnodes}
        # transient per-ply masks (reference compiler.py:112-113, state.py:121-123):
        # three bitboards after the piece-type planes
        self.transient = any(t in types for t in (n.CapturedMask, n.HoppedMask,
                                                   n.PromotedMask))
        self.tbase = self.xbase
        if self.transient:
            self.xbase += 3 * self.W
        # codec / mechanics family (reference compiler.py:212-221): any movement
        # phase makes the movement codec; placement phases then act on cells
        kinds = {type(p.mechanic) for p in spec.phases}
        self.grid = None
        if n.MoveMechanic in kinds:
            self.grid = self._detect_gridworld()
            self.mech_kind = 2 if self.grid is not None else 1
        else:
            self.mech_kind = 0
        self.has_flip = n.FlipEffect in types
        scores = any(t in types for t in (n.ScoreFn, n.SetScoreEffect, n.IncrementScoreEffect))
        scores |= any(isinstance(x, n.CaptureEffect) and x.increment_score for x in allnodes)
        scores |= any(r.result.kind == "by_score" for r in spec.end_rules)
        passing = any(p.force_pass for p in spec.phases) or n.PassedPred in types
        must_move = any(isinstance(x, n.ExtraTurnEffect) and x.same_piece for x in allnodes)
        last_action = any(t in types for t in (      # reference compiler.py:114-116
            n.ActionWasPred, n.CanMoveAgainPred, n.PrevMoveMask, n.LastMoveInPred,
            n.CustodialMask, n.CornerCustodialMask, n.ExtraTurnEffect))
        self.needs_next_count = n.NoLegalActionsPred in types
        for x in allnodes:
            if isinstance(x, n.ConnectedFn):
                self._conn_plan(x)
        # anchored line candidates (reference compiler.py:122-135)
        self.anchor_lines = set()
        cands = []
        if not self.has_flip:
            for rule in spec.end_rules:
                for x in n.walk(rule.condition):
                    if isinstance(x, n.FunctionPred) and isinstance(x.fn, n.LineFn):
                        line = x.fn
                        if line.player != n.MOVER:
                            continue
                        T = len(self.board.line_windows(line.length, line.orientation))
                        if T * line.length > ANCHOR_COST_THRESHOLD:
                            cands.append(line)
        self.phase_mult = len(spec.phases) > 1 or any(p.kind == "once_through"
                                                      for p in spec.phases)
        self.turn_pos = any(len(p.order) != len(set(p.order)) for p in spec.phases)
        self.has_pass = passing
        self.layout = {"scores": scores, "passing": passing, "must_move": must_move,
                       "last_action": last_action or bool(cands),
                       "transient_masks": self.transient, "connectivity": len(self.conn_plans),
                       "phase": self.phase_mult, "turn_pos": self.turn_pos}
        self._anchor_candidates = cands
        self._last_action_base = last_action
        # action codec (reference codec.py:58-69)
        base = {0: self.C, 1: self.C * self.C}.get(self.mech_kind)
        if base is None:
            base = len(self.grid[2])
        self.A = base + (1 if passing else 0)
        self.PASS = base if passing else -1

    def _conn_plan(self, node):
        dirs = resolve_direction(node.directions or ("any",), n.P1, self.forward, self.board)
        if dirs not in self.conn_plans:
            self.conn_plans.append(dirs)
        return self.conn_plans.index(dirs)

    # ------------------------------------------------------------ static masks

    def static_mask(self, node):
        """(C,) bool for geometry-only masks, else None (reference exprs.py:42-88)."""
        t = type(node)
        B = self.board
        if t is n.CenterMask:
            return B.center_mask
        if t is n.CornersMask:
            return B.corners_mask
        if t is n.RowMask:
            return np.asarray(B.row_of == node.index)
        if t is n.ColumnMask:
            return np.asarray(B.col_of == node.index)
        if t is n.EdgeMask and node.which not in ("forward", "backward"):
            return B.edge_masks[node.which]
        if t is n.RegionMask:
            return self.regions[node.region]
        if t is n.MultiMask:
            out = np.zeros(self.C, dtype=bool)
            for m in B.multi_mask(node.kind):
                out |= m
            return out
        if t in (n.MaskAnd, n.MaskOr):
            parts = [self.static_mask(i) for i in node.items]
            if any(p is None for p in parts):
                return None
            out = parts[0].copy()
            for p in parts[1:]:
                out = (out & p) if t is n.MaskAnd else (out | p)
            return out
        if t is n.MaskNot:
            inner = self.static_mask(node.item)
            return None if inner is None else ~inner
        return None

    def _static_union(self, masks):
        out = np.zeros(self.C, dtype=bool)
        for m in masks:
            s = self.static_mask(m)
            if s is None:
                # the reference cannot compile this either (exprs.py:92-97)
                raise UnsupportedConstruct(f"{type(m).__name__} is not static")
            out |= s
        return out

    # ------------------------------------------------------------ expressions
    # All expression code assumes locals: s (state), mover (int), me / op (BBW)

    @staticmethod
    def side(ref):
        if ref in (n.MOVER, ""):
            return "mover"
        if ref == n.OPPONENT:
            return "(1 - mover)"
        if ref in ("P1", 0):
            return "0"
        if ref in ("P2", 1):
            return "1"
        _fail(f"cannot resolve side reference {ref!r}")

    @staticmethod
    def stones(side_expr):
        if side_expr == "mover":
            return "me"
        if side_expr == "(1 - mover)":
            return "op"
        return "s.own0" if side_expr == "0" else "s.own1"

    def mask(self, node):
        st = self.static_mask(node)
        if st is not None:
            return self.em.const(st)
        t = type(node)
        if t is n.EmptyMask:
            return f"lx::andnot({self.em.const(self.valid)}, s.own0 | s.own1)"
        if t is n.OccupiedMask:
            if not node.who:
                return "(s.own0 | s.own1)"
            return self.stones(self.side(node.who))
        if t is n.EdgeMask:              # forward / backward edges per player
            names = []
            for pl in (n.P1, n.P2):
                facing = self.forward.get(pl)
                if facing is None:
                    _fail("edge forward/backward needs set_forward")
                if node.which == "backward":
                    facing = OPPOSITE[facing]
                names.append(self.em.const(self.board.edge_masks[
                    {"up": "top", "down": "bottom", "left": "left", "right": "right"}[facing]]))
            return f"lx::sel(mover != 0, {names[0]}, {names[1]})"
        if t is n.AdjacentMask:
            inner = self.mask(node.inner)
            tmp = self.em.fresh("adj")
            parts = []
            for d1, d2 in direction_pairs(node.directions or ("any",), self.forward, self.board):
                a = self.nb(OPPOSITE[d1], tmp)
                if d1 == d2:
                    parts.append(a)
                else:
                    parts.append(f"lx::sel(mover != 0, {a}, {self.nb(OPPOSITE[d2], tmp)})")
            body = " | ".join(parts)
            return f"([&]() {{ const BBW {tmp} = {inner}; return BBW({body}); }}())"
        if t in (n.MaskAnd, n.MaskOr):
            op = " & " if t is n.MaskAnd else " | "
            return "(" + op.join(self.mask(i) for i in node.items) + ")"
        if t is n.MaskNot:
            return f"lx::andnot({self.em.const(self.valid)}, {self.mask(node.item)})"
        if t is n.CustodialMask:
            if not self.anchored_ctx:
                return self.custodial_global(node)
            return self.custodial_anchored(node)
        if t is n.CornerCustodialMask:
            return self.corner_custodial(node)
        if t is n.LineFn:
            return self.line_mask(node)
        if t in (n.HoppedMask, n.CapturedMask, n.PromotedMask):   # exprs.py:152-165
            k = {n.HoppedMask: 0, n.CapturedMask: 1, n.PromotedMask: 2}[t]
            return self._tplane(k)
        if t is n.PrevMoveMask:                 # reference exprs.py:167-176
            sd = self.side(node.who)
            return (f"([&]() {{ const int d_ = ({sd}) ? s.ldbp1 : s.ldbp0; "
                    f"return d_ >= 0 ? lx::onehot<W>(cell_bit(d_)) : lx::bb_zero<W>(); }}())")
        _fail(f"mask {t.__name__} is not lowered yet")

    def corner_custodial(self, node):
        """Enemy piece on a corner whose two orthogonal neighbours are the
        side's; in effects only when one of them was just moved to by the
        side (reference exprs.py:381-408)."""
        side = self.side(node.mover)
        B = self.board
        corners = []
        for c in B.corner_cells:
            nbrs = [int(B.neighbors[d][c]) for d in ("up", "down", "left", "right")
                    if d in B.neighbors and int(B.neighbors[d][c]) != self.C]
            if len(nbrs) == 2:
                corners.append((c, nbrs[0], nbrs[1]))
        name = f"corner_{self.em.fresh('cc')}"
        tgt = self.piece_filter(node.piece, "tgt")
        lines = []
        for c, n1, n2 in corners:
            b, b1, b2 = (int(self.bit_of[x]) for x in (c, n1, n2))
            cond = f"lx::test(tg, {b}) && lx::test(fl, {b1}) && lx::test(fl, {b2})"
            if self.anchored_ctx:
                cond += f" && (s.last_dest == {n1} || s.last_dest == {n2}) && s.last_mover == side"
            lines.append(f"        if ({cond}) lx::setbit(out, {b});")
        body = "\n".join(lines)
        self.em.helper(name, f"""    static __device__ __forceinline__ BBW {name}(const St& s, int mover) {{
        const int side = {side};
        const BBW fl = side ? s.own1 : s.own0;
        const BBW tgt = side ? s.own0 : s.own1;
        const BBW tg = {tgt};
        BBW out = lx::bb_zero<W>();
{body}
        return out;
    }}""")
        return f"{name}(s, mover)"

    # -- custodial ------------------------------------------------------------

    def custodial_dirs(self, node):
        dirs = []
        for d in self.board.orientation_dirs(node.orientation):
            dirs += [d, OPPOSITE[d]]
        return dirs

    def _ks_fill(self, e, gen, pro, max_run, ind="            "):
        """Kogge-Stone occluded fill along e: g = gen plus every cell y of a
        run y, y+e, .., y+(j-1)e of `pro` cells with y+je in gen, j <= 2^m - 1
        >= max_run.  Log-steps walk(e, 1), walk(e, 2), walk(e, 4) ... with
        exact k-step validity masks (no wrap).  Declares BBW g."""
        if os.environ.get("LX_KS_PREMASK", "1") != "0":
            # the propagator masked once to cells with an e-neighbour: p_k(x)
            # then implies x + k*e is a valid walk (p_2(x) = p(x) & p(x + e)
            # needs both steps valid, and so on), so the log-steps are raw
            # shifts -- one LOP3 per word instead of two (the walk masks)
            S = self._shift[e]
            v1 = self.em.const(self._walk_ok(e, 1))
            code = [f"{ind}BBW g = {gen};", f"{ind}BBW p = {pro} & {v1};"]
            k, covered = 1, 0
            while covered < max_run:
                code.append(f"{ind}g = g | (p & lx::gather<W, {S * k}>(g));")
                covered += k
                if covered < max_run:
                    code.append(f"{ind}p = p & lx::gather<W, {S * k}>(p);")
                k *= 2
            return code
        code = [f"{ind}BBW g = {gen};", f"{ind}BBW p = {pro};"]
        k, covered = 1, 0
        while covered < max_run:
            code.append(f"{ind}g = g | (p & {self.walk(e, k, 'g')});")
            covered += k
            if covered < max_run:
                code.append(f"{ind}p = p & {self.walk(e, k, 'p')};")
            k *= 2
        return code

    # -- cell probes (big boards) --------------------------------------------

    @property
    def use_probe(self):
        """Anchored rules on boards of >= 6 words per side use cell probes
        through the shared-memory mirror instead of whole-board shifts."""
        return self.W >= 6

    # -- row mirror (big placement boards) ------------------------------------
    # Per thread, each player's stones as one 32-bit word per grid row (bit
    # RM_PAD + column) with RM_PAD zero rows above and below and zero columns
    # either side, kept in shared memory and updated at each placement /
    # capture (rebuilt from the registers when a state enters a kernel).  A
    # probe of cell (r + dr, c + dc) is then a row load at a constant offset
    # from row r and a bit test: no bounds checks (off-board cells read the
    # zero padding) and no per-probe address arithmetic.
    RM_PAD = 4

    @property
    def row_mirror_ok(self):
        return (self.use_probe and self.mech_kind == 0 and self.NPL == 0
                and self.emb_cols + 2 * self.RM_PAD <= 32
                and os.environ.get("LX_ROW_MIRROR", "1") != "0")

    def _drdc(self, d):
        S = self._shift[d]
        cols = self.emb_cols
        dr = (S + cols // 2) // cols if S >= 0 else -((-S + cols // 2) // cols)
        return dr, S - dr * cols

    def _rm_code(self):
        """Row-mirror layout constants and maintenance (emitted when used)."""
        if not self.rm_used:
            return ("    static constexpr bool ROW_MIRROR = false;\n"
                    "    static __device__ __forceinline__ void rm_build(const St&) {}\n"
                    "    static __device__ __forceinline__ void rm_set(int, int) {}")
        R, EC, P = self.emb_rows, self.emb_cols, self.RM_PAD
        build = []
        for pl, own in ((0, "s.own0"), (1, "s.own1")):
            for k in range(P):
                build.append(f"        rm_row({pl}, {-1 - k})[0] = 0u; rm_row({pl}, {R + k})[0] = 0u;")
            for r in range(R):
                b0 = r * EC
                wi, sh = b0 >> 5, b0 & 31
                lo = f"{own}.w[{wi}]"
                hi = f"{own}.w[{wi + 1}]" if wi + 1 < self.W else "0u"
                ext = f"__funnelshift_r({lo}, {hi}, {sh})" if sh else lo
                build.append(f"        rm_row({pl}, {r})[0] = ({ext} & 0x{(1 << EC) - 1:x}u) << {P};")
        build = "\n".join(build)
        return f"""    static constexpr bool ROW_MIRROR = true;
    static constexpr int RM_ROWS = {R + 2 * P}, RM_PAD = {P}, RM_COLS = {EC};
    // row `row` (may be negative: padding) of `player`'s plane, this thread's slot
    static __device__ __forceinline__ u32* rm_row(int player, int row) {{
        return lx::RowMirror<RM_ROWS>::slot() + (player * RM_ROWS + row + RM_PAD) * LX_MIRROR_STRIDE;
    }}
    static __device__ __forceinline__ void rm_build(const St& s) {{
{build}
    }}
    static __device__ __forceinline__ void rm_set(int player, int b) {{
        const int r = b / RM_COLS, c = b - r * RM_COLS;
        rm_row(player, r)[0] |= 1u << (c + RM_PAD);
    }}"""

    def capture_rm_block(self, e, ind):
        """Capture effect (effects.py:29-48) with a fixed-length anchored
        custodial mask on the row mirror: the target / flanker rows around the
        anchor are loaded once as windows (bit Q = the anchor's column) and
        every direction is three bit tests; a capture clears its cells in the
        mirror rows and the register board (rare, divergent)."""
        node = e.mask
        if not (type(node) is n.CustodialMask and self.anchored_ctx and self.row_mirror_ok
                and self.piece_mode == "single" and node.length != "any"
                and not self.transient and self._probe_in_mirror(node)):
            return None
        n_len = node.length
        dirs = [self._drdc(d) + (self._shift[d],) for d in self.custodial_dirs(node)]
        if any(abs(dr) * (n_len + 1) > self.RM_PAD or abs(dc) * (n_len + 1) > self.RM_PAD
               for dr, dc, _ in dirs):
            return None
        self.rm_used = True
        Q = max(abs(dc) for dr, dc, _ in dirs) * (n_len + 1)
        side = self.side(node.mover)
        tg_rows = sorted({k * dr for dr, dc, _ in dirs for k in range(1, n_len + 1)})
        sd_rows = sorted({(n_len + 1) * dr for dr, dc, _ in dirs})
        nm = lambda k: f"m{-k}" if k < 0 else f"p{k}"                      # noqa: E731
        lines = [f"        const u32 t_{nm(k)} = rm_row(tg, r + {k})[0] >> sh;" for k in tg_rows]
        lines += [f"        const u32 f_{nm(k)} = rm_row(side, r + {k})[0] >> sh;" for k in sd_rows]
        for dr, dc, S in dirs:
            conds = [f"(t_{nm(k * dr)} >> {Q + k * dc})" for k in range(1, n_len + 1)]
            conds.append(f"(f_{nm((n_len + 1) * dr)} >> {Q + (n_len + 1) * dc})")
            lines.append(f"        if ((" + " & ".join(conds) + ") & 1u) {")
            for k in range(1, n_len + 1):
                lines.append(f"            rm_row(tg, r + {k * dr})[0] &= ~(1u << (col + RM_PAD + {k * dc}));")
                lines.append(f"            if (tg) lx::clearbit(s.own1, c + {k * S}); "
                             f"else lx::clearbit(s.own0, c + {k * S});")
            lines.append(f"            ncap += {n_len};")
            lines.append("        }")
        body = "\n".join(lines)
        name = f"capture_rm_{self.em.fresh('c')}"
        self.em.helper(name, f"""    // mirrored capture probes: returns the number of cells taken
    static __device__ __forceinline__ int {name}(St& s, int mover) {{
        const int side = {side};
        const int tg = 1 - side;
        if (!(s.last_dest >= 0 && s.last_mover == side)) return 0;
        const int c = cell_bit(s.last_dest);
        const int r = c / {self.emb_cols};
        const int col = c - r * {self.emb_cols};
        const int sh = col + RM_PAD - {Q};        // window bit {Q} = the anchor's column
        int ncap = 0;
{body}
        return ncap;
    }}""")
        inc = ""
        if e.increment_score:
            inc = f" if (mover) s.sc1 += g; else s.sc0 += g;"
        return f"{ind}{{ const int g = {name}(s, mover);{inc} (void)g; }}"

    def line_rm_probe(self, node):
        """Anchored line test (exprs.py:484-535) on the row mirror: the rows
        around the anchor are loaded once as windows (bit P = the anchor's
        column) and the run along each axis is counted from bit tests."""
        if not self.row_mirror_ok or node.exclude is not None or self.piece_mode != "single":
            return None
        L = node.length
        P = L if node.exact else L - 1
        axes = []
        for d in self.board.orientation_dirs(node.orientation):
            a = self._drdc(d)
            b = self._drdc(OPPOSITE[d])
            axes.append((a, b))
        if any(abs(x) * P > self.RM_PAD for (a, b) in axes for x in a + b):
            return None
        self.rm_used = True
        side = self.side(node.player)
        rows = sorted({k * dr for (a, b) in axes for (dr, dc) in (a, b) for k in range(0, P + 1)})
        nm = lambda k: f"m{-k}" if k < 0 else f"p{k}"                      # noqa: E731
        Q = max(abs(dc) for (a, b) in axes for (dr, dc) in (a, b)) * P
        lines = [f"        const u32 w_{nm(k)} = rm_row(side, r + {k})[0] >> sh;" for k in rows]
        lines.append(f"        if (!((w_p0 >> {Q}) & 1u)) return false;")
        for (a, b) in axes:
            lines.append("        {")
            lines.append("            int run = 0;")
            for (dr, dc) in (a, b):
                lines.append("            { u32 on = 1u;")
                for k in range(1, P + 1):
                    lines.append(f"              on &= w_{nm(k * dr)} >> {Q + k * dc}; run += on & 1u;")
                lines.append("            }")
            lines.append(f"            if (run {'==' if node.exact else '>='} {L - 1}) return true;")
            lines.append("        }")
        body = "\n".join(lines)
        name = f"line_rm_{self.em.fresh('a')}"
        self.em.helper(name, f"""    static __device__ __forceinline__ bool {name}(const St& s, int mover) {{
        const int side = {side};
        if (!(s.last_dest >= 0 && s.last_mover == mover)) return false;
        const int c = cell_bit(s.last_dest);
        const int r = c / {self.emb_cols};
        const int col = c - r * {self.emb_cols};
        const int sh = col + RM_PAD - {Q};        // window bit {Q} = the anchor's column
{body}
        return false;
    }}""")
        return f"{name}(s, mover)"

    def _bitmap_code(self):
        """cell id <-> bit position maps (identity on row-major boards)."""
        if self.ident:
            return ("    static __device__ __forceinline__ int cell_bit(int c) { return c; }\n"
                    "    static __device__ __forceinline__ int bit_cell(int b) { return b; }")
        cell_of = np.full(self.NB, -1, dtype=np.int64)
        cell_of[self.bit_of] = np.arange(self.C)
        cb = ", ".join(str(int(x)) for x in self.bit_of)
        bc = ", ".join(str(int(x)) for x in cell_of)
        return (f"    static __device__ __forceinline__ int cell_bit(int c) {{\n"
                f"        static __device__ const short t[{self.C}] = {{{cb}}};\n"
                f"        return t[c];\n    }}\n"
                f"    static __device__ __forceinline__ int bit_cell(int b) {{\n"
                f"        static __device__ const short t[{self.NB}] = {{{bc}}};\n"
                f"        return t[b];\n    }}")

    def _max_steps(self, d):
        """Expression: how many steps along d stay inside the bit grid from
        (r, col) of the anchor's bit (embedded grid for hexagons: cells outside
        the hexagon are padding bits that are never set)."""
        S = self._shift[d]
        cols = self.emb_cols
        dr = (S + cols // 2) // cols if S >= 0 else -((-S + cols // 2) // cols)
        dc = S - dr * cols
        terms = []
        if dr > 0:
            terms.append(f"({self.emb_rows - 1} - r) / {dr}")
        elif dr < 0:
            terms.append(f"r / {-dr}")
        if dc > 0:
            terms.append(f"({cols - 1} - col) / {dc}")
        elif dc < 0:
            terms.append(f"col / {-dc}")
        if not terms:
            return "0"
        out = terms[0]
        for t in terms[1:]:
            out = f"lx::imin({out}, {t})"
        return out

    def _probe_in_mirror(self, node):
        """Captured cells can be removed from the mirrored target plane as they
        are found when no direction probes a cell another direction captures:
        k*S_e != j*S_d for 1 <= k <= n+1, 1 <= j <= n."""
        n_len = node.length
        dirs = self.custodial_dirs(node)
        steps = {d: self._shift[d] for d in dirs}
        return all(k * steps[e] != j * steps[d] for d in dirs for e in dirs if d != e
                   for k in range(1, n_len + 2) for j in range(1, n_len + 1))

    def capture_probe_block(self, e, ind):
        """Capture effect (reference effects.py:29-48) whose mask is a probed
        anchored custodial run with the cells kept in the mirror: the probes
        clear captured cells from the mirrored target plane and count them,
        and only a lane that captured copies that plane back to its register
        board -- instead of diffing and clearing every word of both boards
        each ply (Pente: captures are rare).  None when not applicable."""
        node = e.mask
        if os.environ.get("LX_CAPTURE_FAST", "1") == "0":       # A/B switch
            return None
        if not (type(node) is n.CustodialMask and self.anchored_ctx and
                self.piece_mode == "single" and self.use_probe and node.length != "any"
                and not self.transient and self.NPL == 0 and self._probe_in_mirror(node)):
            return None
        side = self.side(node.mover)
        n_len = node.length
        name = f"capture_probe_{self.em.fresh('c')}"
        lines = []
        for d in self.custodial_dirs(node):
            S = self._shift[d]
            lines.append(f"        {{ const bool ok = {self._max_steps(d)} >= {n_len + 1};")
            conds = [f"M::probe_if(ok, tg, c + {k * S})" for k in range(1, n_len + 1)]
            conds.append(f"M::probe_if(ok, side, c + {(n_len + 1) * S})")
            lines.append("        if (" + " & ".join(conds) + ") {")
            for k in range(1, n_len + 1):
                lines.append(f"            M::clear(tg, c + {k * S});")
            lines.append(f"            ncap += {n_len};")
            lines.append("        } }")
        body = "\n".join(lines)
        self.em.helper(name, f"""    // probes + mirror clears of a capture; returns the number of cells taken
    static __device__ __forceinline__ int {name}(St& s, int mover) {{
        typedef lx::Mirror<W> M;
        const int side = {side};
        const int tg = 1 - side;
        int ncap = 0;
        if (!(s.last_dest >= 0 && s.last_mover == side)) return 0;
        M::store(s.own0, s.own1);
        s.mirror_fresh = 1;
        const int c = cell_bit(s.last_dest);
        const int r = c / {self.emb_cols};
        const int col = c - r * {self.emb_cols};
{body}
        if (ncap) {{                       // rare: the target plane comes back from the mirror
            const BBW pl = M::load(tg);
            if (tg) s.own1 = pl; else s.own0 = pl;
        }}
        return ncap;
    }}""")
        inc = ""
        if e.increment_score:
            inc = f" if (mover) s.sc1 += g; else s.sc0 += g;"
        return f"{ind}{{ const int g = {name}(s, mover);{inc} (void)g; }}"

    def custodial_anchored_probe(self, node):
        """Fixed-length anchored custodial run by probing cells from last_dest:
        anchor+kd (k=1..n) target stones and anchor+(n+1)d a flanker
        (reference exprs.py:254-292 with length n)."""
        side = self.side(node.mover)
        n_len = node.length
        name = f"custodial_probe_{self.em.fresh('c')}"
        lines = []
        dirs = self.custodial_dirs(node)
        # captured cells are removed from the mirrored target plane as they are
        # found (result = registers minus mirror) when no direction probes a
        # cell another direction captures; otherwise cells are set in a
        # register bitboard
        in_mirror = self._probe_in_mirror(node)
        for d in dirs:
            S = self._shift[d]
            # branch-free: all probes issue (clamped when off-board), one rare branch
            lines.append(f"        {{ const bool ok = {self._max_steps(d)} >= {n_len + 1};")
            conds = [f"M::probe_if(ok, tg, c + {k * S})" for k in range(1, n_len + 1)]
            conds.append(f"M::probe_if(ok, side, c + {(n_len + 1) * S})")
            lines.append("        if (" + " & ".join(conds) + ") {")
            for k in range(1, n_len + 1):
                lines.append(f"            M::clear(tg, c + {k * S});" if in_mirror else
                             f"            lx::setbit(out, c + {k * S});")
            lines.append("        } }")
        body = "\n".join(lines)
        ret = ("lx::andnot(lx::sel(tg != 0, s.own0, s.own1), M::load(tg))" if in_mirror else "out")
        self.em.helper(name, f"""    static __device__ __forceinline__ BBW {name}(const St& s, int mover) {{
        typedef lx::Mirror<W> M;
        const int side = {side};
        const int tg = 1 - side;
        BBW out = lx::bb_zero<W>();
        if (!(s.last_dest >= 0 && s.last_mover == side)) return out;
        M::store(s.own0, s.own1);
        const int c = cell_bit(s.last_dest);
        const int r = c / {self.emb_cols};
        const int col = c - r * {self.emb_cols};
{body}
        return {ret};
    }}""")
        return f"{name}(s, mover)"

    def custodial_anchored_rays(self, node):
        """Anchored custodial runs of any length on boards of <= 64 cells with
        per-cell ray masks (reference exprs.py:254-292): along each direction
        the first non-target cell on the ray from the anchor is found with a
        lowest/highest-set-bit trick; the run is flanked iff that cell is a
        flanker, and the run is every ray cell before it."""
        side = self.side(node.mover)
        name = f"custodial_rays_{self.em.fresh('c')}"
        dirs = self.custodial_dirs(node)
        C = self.C
        rows = []
        for d in dirs:
            nt = self.board.neighbors[d]
            vals = []
            for c in range(C):
                m, x = 0, int(nt[c])
                while x != C:
                    m |= 1 << int(self.bit_of[x])
                    x = int(nt[x])
                vals.append(m)
            rows.append("{" + ", ".join(f"0x{v:016x}ull" for v in vals) + "}")
        table = f"RAYS_{name}"
        self.em.helper(table, f"    static __device__ __forceinline__ u64 {table}(int d, int c) {{\n"
                              f"        static __device__ const u64 t[{len(dirs)}][{C}] = {{\n            "
                              + ",\n            ".join(rows) + "};\n        return t[d][c];\n    }")
        lines = []
        for k, d in enumerate(dirs):
            S = self._shift[d]
            lines.append("        {")
            lines.append(f"            const u64 r = {table}({k}, c);")
            lines.append("            const u64 blk = r & ~tgt;            // first of these ends the run")
            if S > 0:
                lines.append("            const u64 first = blk & (0ull - blk);")
                lines.append("            if (first & flank) run |= r & (first - 1ull);")
            else:
                lines.append("            const u64 first = blk ? (1ull << (63 - __clzll((long long)blk))) : 0ull;")
                lines.append("            if (first & flank) run |= r & ~((first << 1) - 1ull);")
            lines.append("        }")
        body = "\n".join(lines)
        W = self.W
        to64 = "(u64)b.w[0]" + (" | ((u64)b.w[1] << 32)" if W == 2 else "")
        self.em.helper(name, f"""    static __device__ __forceinline__ u64 {name}_u64(const BBW& b) {{ return {to64}; }}
    static __device__ __forceinline__ BBW {name}(const St& s, int mover) {{
        const int side = {side};
        BBW out = lx::bb_zero<W>();
        if (!(s.last_dest >= 0 && s.last_mover == side)) return out;
        const u64 flank = {name}_u64(side ? s.own1 : s.own0);
        const u64 tgt = {name}_u64(side ? s.own0 : s.own1);
        const int c = s.last_dest;
        u64 run = 0ull;
{body}
        out.w[0] = (u32)run;
        {"out.w[1] = (u32)(run >> 32);" if W == 2 else ""}
        return out;
    }}""")
        return f"{name}(s, mover)"

    def line_anchored_probe(self, node):
        """Anchored line test (reference exprs.py:484-535) by probing: the run
        of the player's stones through last_dest along some axis has at least
        `length` cells."""
        rm = self.line_rm_probe(node)
        if rm is not None:
            return rm
        if node.exclude is not None or self.piece_mode != "single":
            _fail("probed line with exclude: / several piece types is not lowered yet")
        side = self.side(node.player)
        L = node.length
        name = f"line_probe_{self.em.fresh('a')}"
        lines = []
        steps = L if node.exact else L - 1          # exact: detect overlines too
        for d in self.board.orientation_dirs(node.orientation):
            for sgn, dd in ((1, d), (-1, OPPOSITE[d])):
                S = self._shift[dd]
                lines.append(f"        {{ const int mk = {self._max_steps(dd)}; u32 on = 1u;")
                for k in range(1, steps + 1):
                    lines.append(f"          on &= M::probe_if(mk >= {k}, side, c + {k * S}); "
                                 f"run += on;")
                lines.append("        }")
            lines.append(f"        if (run {'==' if node.exact else '>='} {L - 1}) return true;")
            lines.append("        run = 0;")
        body = "\n".join(lines)
        self.em.helper(name, f"""    static __device__ __forceinline__ bool {name}(const St& s, int mover) {{
        typedef lx::Mirror<W> M;
        const int side = {side};
        if (!(s.last_dest >= 0 && s.last_mover == mover)) return false;
        const int c = cell_bit(s.last_dest);
        // only the player's stones are probed; a capture probe earlier in this
        // ply left the mirror current (captures change the other plane only)
        if (!s.mirror_fresh) M::store_plane(side, s.own0, s.own1);
        if (!M::probe(side, c)) return false;
        const int r = c / {self.emb_cols};
        const int col = c - r * {self.emb_cols};
        int run = 0;
{body}
        return false;
    }}""")
        return f"{name}(s, mover)"

    def custodial_anchored(self, node):
        """Anchored custodial runs from last_dest (reference exprs.py:254-292).

        For each walk direction, the run of target stones that starts next to
        the anchor is kept when the next cell is a flanker; ``length`` fixes
        the run length.  The reference bounds runs by the padded ray length
        L (runlen < L), which any flanked run on the board satisfies.
        """
        if self.piece_mode == "single" and self.use_probe and node.length != "any":
            return self.custodial_anchored_probe(node)
        if self.piece_mode == "single" and node.length == "any" and self.W <= 2:
            return self.custodial_anchored_rays(node)
        side = self.side(node.mover)
        name = f"custodial_{self.em.fresh('c')}"
        lines = []
        for d in self.custodial_dirs(node):
            steps = self.board.ray_length(d) - 1 if node.length == "any" else node.length
            steps = max(steps, 0)
            if steps == 0:
                continue
            lines.append("        {")
            if node.length == "any":
                # run of targets from the anchor along d (fill moves forward: opposite gather)
                lines += self._ks_fill(OPPOSITE[d], "a", "tgt", steps)
                lines.append("            const BBW run = g & tgt;")
            else:
                lines.append("            BBW x = " + self.nb(OPPOSITE[d], "a") + " & tgt;")
                lines.append("            BBW run = x;")
                for _ in range(steps - 1):
                    lines.append("            x = " + self.nb(OPPOSITE[d], "x") + " & tgt;")
                    lines.append("            run = run | x;")
            check = ""
            if node.length != "any":
                check = f" && lx::popc(run) == {node.length}"
            lines.append("            const bool ok = lx::any(" + self.nb(OPPOSITE[d], "run")
                         + f" & flank){check};")
            lines.append("            out = lx::sel(ok, out, out | run);")
            lines.append("        }")
        body = "\n".join(lines)
        code = f"""    static __device__ __forceinline__ BBW {name}(const St& s, int mover) {{
        const int side = {side};
        const BBW flank = side ? s.own1 : s.own0;
        const BBW tgt = {self.piece_filter(node.piece, "(side ? s.own0 : s.own1)")};
        BBW out = lx::bb_zero<W>();
        if (!(s.last_dest >= 0 && s.last_mover == side)) return out;
        const BBW a = lx::onehot<W>(cell_bit(s.last_dest));
{body}
        return out;
    }}"""
        self.em.helper(name, code)
        return f"{name}(s, mover)"

    def result_sim(self, pred, cand, write_stmt):
        """Placement result predicate by simulation (reference
        PlacementMechanics._simulate, mechanics.py:445-461): for every
        candidate cell, place on a copy of the state (transient masks
        cleared, last-action fields and reach sets updated as by a real
        placement) and evaluate the predicate in the anchored context."""
        name = f"result_sim_{self.em.fresh('r')}"
        self.anchored_ctx = True
        try:
            cond = self.predicate(pred)
        finally:
            self.anchored_ctx = False
        self.em.helper(name, f"""    static __device__ __forceinline__ bool {name}_p(const St& s, int mover) {{
        const BBW me = mover ? s.own1 : s.own0;
        const BBW op = mover ? s.own0 : s.own1;
        (void)me; (void)op;
        return {cond};
    }}
    static __device__ __forceinline__ BBW {name}(const St& s, const BBW& cand) {{
        const int mover = s.cur;
        BBW out = lx::bb_zero<W>();
        for (int w = 0; w < W; w++) {{
            u32 bits = cand.w[w];
            while (bits) {{
                const int b = 32 * w + __ffs(bits) - 1;
                bits &= bits - 1u;
                St t = s;
                clear_transient(t);
                {write_stmt}
                if ({name}_p(t, mover)) lx::setbit(out, b);
            }}
        }}
        return out;
    }}""")
        return f"{name}(s, {cand})"

    def custodial_global(self, node):
        """Every flanked target run on the board (reference
        mask_custodial_global, exprs.py:294-319): a target cell is marked when
        its maximal target run along an axis is bounded by the side's pieces
        at both ends (any length), or for a fixed length n when that run has
        exactly n cells.  Runs reaching the board edge are never flanked."""
        side = self.side(node.mover)
        name = f"custodial_global_{self.em.fresh('g')}"
        lines = []
        for d in self.board.orientation_dirs(node.orientation):
            e = OPPOSITE[d]
            lines.append("        {")
            if node.length == "any":
                ray = max(self.board.ray_length(d), 1)
                lines += self._ks_fill(d, "flank", "tgt", ray, ind="            ")
                lines.append("            const BBW fwd = g & tgt;")
                lines.append("        {")
                lines += self._ks_fill(e, "flank", "tgt", ray, ind="            ")
                lines.append("            out = out | (fwd & g & tgt);")
                lines.append("        }")
            else:
                n_len = int(node.length)
                for dd in (d,):                  # the inverse walk marks the same runs
                    od = OPPOSITE[dd]
                    conds = [f"{self.nb(od, 'flank')}", "tgt"]
                    for k in range(1, n_len):
                        conds.append(self.walk(dd, k, "tgt"))
                    conds.append(self.walk(dd, n_len, "flank"))
                    lines.append("            {")
                    lines.append(f"                const BBW st = {' & '.join(conds)};")
                    marks = ["st"] + [self.walk(od, k, "st") for k in range(1, n_len)]
                    lines.append(f"                out = out | {' | '.join(marks)};")
                    lines.append("            }")
            lines.append("        }")
        body = "\n".join(lines)
        self.em.helper(name, f"""    static __device__ __forceinline__ BBW {name}(const St& s, int mover) {{
        const int side = {side};
        const BBW flank = side ? s.own1 : s.own0;
        const BBW tgt = {self.piece_filter(node.piece, "(side ? s.own0 : s.own1)")};
        BBW out = lx::bb_zero<W>();
{body}
        return out;
    }}""")
        return f"{name}(s, mover)"

    def would_custodial(self, node):
        """Placement-result fast path (reference exprs.py:334-378): cells whose
        placement would flank a run, computed on the pre-placement board by
        shift composition: z_k[x] = target on x..x+(k-1)d and flanker at x+kd."""
        side = self.side(node.mover)
        name = f"would_{self.em.fresh('w')}"
        max_len = max(max(self.board.ray_length(d) for d in self.custodial_dirs(node)), 1)
        lines = []
        for d in self.custodial_dirs(node):
            lines.append("        {")
            if node.length == "any":
                # cells y of target runs that reach a flanker along d
                lines += self._ks_fill(d, "flank", "tgt", max_len - 1)
                lines.append("            const BBW acc = g & tgt;")
            else:
                lines.append("            BBW z = tgt & " + self.nb(d, "flank") + ";")
                for _ in range(node.length - 1):
                    lines.append("            z = tgt & " + self.nb(d, "z") + ";")
                lines.append("            const BBW acc = z;")
            lines.append("            out = out | " + self.nb(d, "acc") + ";")
            lines.append("        }")
        body = "\n".join(lines)
        code = f"""    static __device__ __forceinline__ BBW {name}(const St& s, int mover) {{
        const int side = {side};
        const BBW flank = side ? s.own1 : s.own0;
        const BBW tgt = {self.piece_filter(node.piece, "(side ? s.own0 : s.own1)")};
        BBW out = lx::bb_zero<W>();
{body}
        return out;
    }}"""
        self.em.helper(name, code)
        return f"{name}(s, mover)"

    # -- lines ------------------------------------------------------------

    def _line_axis(self, L, d):
        """Code computing r = window-start bitmap of L stones of ``b`` along d,
        by doubling r(a+b) = r(a) & walk_a(r(b)) (reference _LineTables.satisfied,
        exprs.py:433-450, as bit-parallel shifts)."""
        have = {1: "b"}
        code = []
        k = 1
        while k * 2 <= L:
            nm = f"r{2 * k}"
            code.append(f"            const BBW {nm} = {have[k]} & {self.walk(d, k, have[k])};")
            have[2 * k] = nm
            k *= 2
        cur_len, cur = k, have[k]
        rest = L - k
        while rest > 0:
            p = 1
            while p * 2 <= rest:
                p *= 2
            nm = f"r{cur_len + p}"
            code.append(f"            const BBW {nm} = {cur} & {self.walk(d, cur_len, have[p])};")
            cur, cur_len, rest = nm, cur_len + p, rest - p
        return code, cur

    def _line_excluded(self, node):
        """Static cells a window may not touch (reference exprs.py:427-431)."""
        ex = node.exclude if isinstance(node.exclude, tuple) else (node.exclude,)
        return self._static_union(ex)

    def _line_fn(self, node, kind):
        excl = self._line_excluded(node) if node.exclude is not None else None
        axes = self.board.orientation_dirs(node.orientation)
        name = f"line_{kind}_{self.em.fresh('l')}"
        body = []
        for d in axes:
            code, r = self._line_axis(node.length, d)
            body.append("        {")
            body += code
            if node.exact:
                # exact: the cells just before and after the window are not the
                # player's (reference exprs.py:444-448; off-board counts as not)
                code.append("")
                body.append(f"            const BBW rx = lx::andnot(lx::andnot({r}, "
                            f"{self.nb(OPPOSITE[d], 'b')}), {self.walk(d, node.length, 'b')});")
                r = "rx"
            if excl is not None:
                allowed = np.zeros(self.C, dtype=bool)
                for dd, cells in self.board.line_windows(node.length, d):
                    if not excl[list(cells)].any():
                        allowed[cells[0]] = True
                r = f"({r} & {self.em.const(allowed)})"
            body.append(f"            acc = acc | {r};" if kind == "any"
                        else f"            acc += lx::popc({r});")
            body.append("        }")
        init = "BBW acc = lx::bb_zero<W>();" if kind == "any" else "int acc = 0;"
        ret = "lx::any(acc)" if kind == "any" else "acc"
        rtype = "bool" if kind == "any" else "int"
        self.em.helper(name, f"""    static __device__ __forceinline__ {rtype} {name}(const BBW& b) {{
        {init}
{chr(10).join(body)}
        return {ret};
    }}""")
        return name

    def line_mask(self, node):
        """Cells of satisfied windows (reference _compile_line_mask,
        exprs.py:468-481): every window-start bit spread over its L cells."""
        stones = self.piece_filter(node.piece, self.stones(self.side(node.player)))
        excl = self._line_excluded(node) if node.exclude is not None else None
        name = f"line_mask_{self.em.fresh('m')}"
        body = []
        for d in self.board.orientation_dirs(node.orientation):
            code, r = self._line_axis(node.length, d)
            body.append("        {")
            body += code
            if node.exact:
                body.append(f"            const BBW rx = lx::andnot(lx::andnot({r}, "
                            f"{self.nb(OPPOSITE[d], 'b')}), {self.walk(d, node.length, 'b')});")
                r = "rx"
            if excl is not None:
                allowed = np.zeros(self.C, dtype=bool)
                for _, cells in self.board.line_windows(node.length, d):
                    if not excl[list(cells)].any():
                        allowed[cells[0]] = True
                r = f"({r} & {self.em.const(allowed)})"
            body.append(f"            const BBW st = {r};")
            parts = ["st"] + [self.walk(OPPOSITE[d], k, "st") for k in range(1, node.length)]
            body.append(f"            acc = acc | {' | '.join(parts)};")
            body.append("        }")
        self.em.helper(name, f"""    static __device__ __forceinline__ BBW {name}(const BBW& b) {{
        BBW acc = lx::bb_zero<W>();
{chr(10).join(body)}
        return acc;
    }}""")
        return f"{name}({stones})"

    def pattern_count(self, node):
        """Number of placements of an offset pattern owned by the player
        (reference _compile_pattern, exprs.py:599-626; placements from
        topology.pattern_table: all distinct rotations with rotate:true).
        Per normalised variant: anchors with a full placement (constant
        mask, exclusions applied) AND the player's stones gathered at each
        offset's constant bit shift; count = sum of popcounts (placements of
        distinct variants are distinct cell sets)."""
        B = self.board
        if node.shape is not None:
            offs = list(Board(node.shape).coords)
        else:
            offs = [(i // node.width, i % node.width) for i in node.offsets]
        if not offs:
            _fail("empty pattern")

        def norm(o):
            amin = min(a for a, _ in o)
            bmin = min(b for _, b in o)
            return tuple(sorted(set((a - amin, b - bmin) for a, b in o)))
        variants = {norm(offs)}
        if node.rotate:
            cur = offs
            hexish = B.kind in ("hexagon", "hex_rectangle")
            for _ in range((6 if hexish else 4) - 1):
                cur = [(-b, a + b) for a, b in cur] if hexish else [(b, -a) for a, b in cur]
                variants.add(norm(cur))
        excl = None
        if node.exclude is not None:
            ex = node.exclude if isinstance(node.exclude, tuple) else (node.exclude,)
            excl = self._static_union(ex)
        stones = self.piece_filter(node.piece, self.stones(self.side(node.player)))
        terms = []
        for var in sorted(variants):
            anchors = np.zeros(self.C, dtype=bool)
            shifts = {}
            for x, (a, b) in enumerate(B.coords):
                cells = []
                for da, db in var:
                    j = B.cell_at((a + da, b + db))
                    if j is None:
                        break
                    cells.append(j)
                if len(cells) != len(var):
                    continue
                if excl is not None and excl[cells].any():
                    continue
                anchors[x] = True
                for (da, db), j in zip(var, cells):
                    shifts.setdefault((da, db), set()).add(int(self.bit_of[j]) - int(self.bit_of[x]))
            if not anchors.any():
                continue
            if any(len(v) != 1 for v in shifts.values()):
                _fail("pattern offsets are not constant bit shifts on this board")
            parts = [self.em.const(anchors)]
            for (da, db) in var:
                S = shifts[(da, db)].pop()
                parts.append(f"lx::gather<W, {S}>(pb)")
            terms.append(f"lx::popc({' & '.join(parts)})")
        if not terms:
            return "0"
        name = f"pattern_{self.em.fresh('p')}"
        self.em.helper(name, f"""    static __device__ __forceinline__ int {name}(const BBW& pb) {{
        return {' + '.join(terms)};
    }}""")
        return f"{name}({stones})"

    def line_exists(self, node):
        """Any window of `length` stones of the player (one axis live at a time)."""
        stones = self.piece_filter(node.piece, self.stones(self.side(node.player)))
        return f"{self._line_fn(node, 'any')}({stones})"

    def line_count(self, node):
        """Number of satisfied windows (LineFn as a function, exprs.py:454-459)."""
        stones = self.piece_filter(node.piece, self.stones(self.side(node.player)))
        return f"{self._line_fn(node, 'count')}({stones})"

    def line_anchored_exists(self, node):
        """Exact anchored form: a satisfied window through last_dest
        (reference exprs.py:484-535) <=> the run of the mover's stones through
        the anchor along some axis has >= length cells."""
        stones = self.piece_filter(node.piece, self.stones(self.side(node.player)))
        L = node.length
        name = f"line_anchor_{self.em.fresh('a')}"
        extra = ""
        if node.exclude is not None:
            ex = self.em.const(self._line_excluded(node))
            if node.exact:
                # the window is the maximal run itself: exactly L cells, none excluded
                extra = f" && !lx::any((e | a) & {ex})"
            else:
                # a window avoiding excluded cells <=> a run of >= L owned
                # non-excluded cells through the anchor
                stones = f"lx::andnot({stones}, {ex})"
        lines = []
        # exact lines need the maximal run through the anchor to be exactly L:
        # grow L steps each way and compare (reference exprs.py:525-533)
        steps = L if node.exact else L - 1
        test = f"== {L}" if node.exact else f">= {L}"
        for d in self.board.orientation_dirs(node.orientation):
            lines.append("        {")
            lines.append("            BBW e = a;")
            for _ in range(steps):
                lines.append(f"            e = (e | {self.nb(d, 'e')} | {self.nb(OPPOSITE[d], 'e')}) & b;")
            lines.append(f"            hit = hit || (lx::popc(e | a) {test}{extra});")
            lines.append("        }")
        body = "\n".join(lines)
        self.em.helper(name, f"""    static __device__ __forceinline__ bool {name}(const St& s, int mover, const BBW& b) {{
        if (!(s.last_dest >= 0 && s.last_mover == mover)) return false;
        const BBW a = lx::onehot<W>(cell_bit(s.last_dest));
        if (!lx::any(a & b)) return false;
        bool hit = false;
{body}
        return hit;
    }}""")
        return f"{name}(s, mover, {stones})"

    # -- connectivity ------------------------------------------------------

    def _conn_targets(self, node):
        if isinstance(node.masks, n.MultiMask):
            targets = self.board.multi_mask(node.masks.kind)
        else:
            targets = [self.static_mask(m) for m in node.masks]
            if any(t is None for t in targets):
                bad = next(m for m, t in zip(node.masks, targets) if t is None)
                raise UnsupportedConstruct(f"{type(bad).__name__} is not static")
        return targets

    def _dilate(self, plan, var, ty="BBW"):
        """Expression: cells with a plan-direction neighbour in `var`.

        Directions that are the composition of two others (nbr_d = nbr_b
        after nbr_a, on every cell, validity included) share a shift:
        x(nbr_d(y)) = nb_a(nb_b(x))(y), so nb_a(x) | nb_a(nb_b(x)) = nb_a(x | nb_b(x)).
        Hex's 6-neighbourhood then costs 4 shifts, the square 8-neighbourhood 4."""
        B = self.board
        C = self.C
        comp = {}
        plan = list(plan)
        for d in plan:
            for a in plan:
                for b in plan:
                    if len({a, b, d}) < 3 or d in comp:
                        continue
                    na, nb_, nd = B.neighbors[a], B.neighbors[b], B.neighbors[d]
                    ok = all((nb_[nd_a] if (nd_a := na[y]) != C else C) == nd[y]
                             for y in range(C))
                    if ok:
                        comp[d] = (a, b)
        base = [d for d in plan if d not in comp or comp[d][0] in comp or comp[d][1] in comp]
        comp = {d: ab for d, ab in comp.items() if d not in base}
        if not comp:
            return " | ".join(self.nb(d, var) for d in plan)
        tmp = {d: f"{var}_{d}" for d in base}
        terms, used = [], set()
        for a in base:
            inner = [tmp[b] for d, (a2, b) in comp.items() if a2 == a]
            if inner:
                used.update(inner)
                terms.append(self.nb(a, f"({var} | {' | '.join(sorted(set(inner)))})"))
            else:
                used.add(tmp[a])
                terms.append(tmp[a])
        decl = " ".join(f"const {ty} {tmp[d]} = {self.nb(d, var)};" for d in base
                        if tmp[d] in used)
        return f"([&]() {{ {decl} return {ty}({' | '.join(terms)}); }}())"

    def _conn_tracking(self):
        """Decide which (connected node, side) pairs get an incrementally
        maintained reach set R = the side's stones connected to target 0.

        Valid when stones are only ever added (placement, no capture/flip):
        components then only grow and merge, so R changes only when a placed
        stone touches target 0 or R, and then grows by exactly the stones
        reachable from it outside R.  Sides are narrowed by (mover_is P)
        conjunctions around the connected test (Hex: P1 top-bottom, P2
        left-right), so Hex keeps 2 sets of 4 words."""
        self.conn_slots = {}
        self.slot_info = []
        types = {type(x) for x in n.walk(self.spec)}
        if (n.CaptureEffect in types or n.FlipEffect in types or not self.conn_plans
                or self.mech_kind != 0):
            return

        def register(node, gate):
            who = node.mover
            if who in (n.MOVER, ""):
                sides = [gate] if gate is not None else [0, 1]
            elif who == n.OPPONENT:
                sides = [1 - gate] if gate is not None else [0, 1]
            elif who in ("P1", 0):
                sides = [0]
            elif who in ("P2", 1):
                sides = [1]
            else:
                sides = [0, 1]
            if len(self._conn_targets(node)) != 2:
                return                      # no reach set: per-component flood test
            for sd in sides:
                key = (id(node), sd)
                if key not in self.conn_slots:
                    self.conn_slots[key] = len(self.slot_info)
                    plan = self.conn_plans[self._conn_plan(node)]
                    self.slot_info.append((sd, self._conn_targets(node), plan))

        def visit(node, gate):
            if isinstance(node, n.PredAnd):
                g = gate
                for it in node.items:
                    if isinstance(it, n.MoverIsPred):
                        g = int(it.player)
                for it in node.items:
                    visit(it, g)
            elif isinstance(node, n.FunctionPred) and isinstance(node.fn, n.ConnectedFn):
                register(node.fn, gate)
            else:
                for ch in node.children():
                    visit(ch, None)

        for rule in self.spec.end_rules:
            visit(rule.condition, None)
        for x in n.walk(self.spec):
            if isinstance(x, n.ConnectedFn) and not any(k[0] == id(x) for k in self.conn_slots):
                register(x, None)

    def _slot_get(self, k):
        W, X = self.W, self.xbase
        words = ", ".join(f"s.ext[{X + k * W + i}]" for i in range(W))
        return f"BBW{{{{{words}}}}}"

    def _slot_set(self, k, var):
        W, X = self.W, self.xbase
        return " ".join(f"s.ext[{X + k * W + i}] = {var}.w[{i}];" for i in range(W))

    def connected(self, node):
        """Some component of the side's stones touches every target mask
        (reference exprs.py:629-652, labels from connectivity.py)."""
        plan = self.conn_plans[self._conn_plan(node)]
        targets = self._conn_targets(node)
        if len(targets) != 2:
            return self._connected_multi(node, plan, targets)
        t0, t1 = self.em.const(targets[0]), self.em.const(targets[1])
        slots = {sd: k for (nid, sd), k in self.conn_slots.items() if nid == id(node)}
        if slots:
            # incremental reach sets: O(1) test
            sd = self.side(node.mover)
            parts = {p: f"lx::any({self._slot_get(k)} & {t1})" for p, k in slots.items()}
            if len(parts) == 1:
                return next(iter(parts.values()))
            return f"(({sd}) ? {parts[1]} : {parts[0]})"
        stones = self.stones(self.side(node.mover))
        dil_f, dil_g = self._dilate(plan, "f"), self._dilate(plan, "g")
        name = f"connected_{self.em.fresh('k')}"
        self.em.helper(name, f"""    static __device__ __forceinline__ bool {name}(const BBW& mine) {{
        // flood the stones reachable from target 0, then test target 1
        BBW f = mine & {t0};
        if (!lx::any(f) || !lx::any(mine & {t1})) return false;
        while (true) {{
            BBW g = (f | {dil_f}) & mine;
            g = (g | {dil_g}) & mine;
            if (lx::equal(g, f)) break;
            f = g;
        }}
        return lx::any(f & {t1});
    }}""")
        return f"{name}({stones})"

    def _connected_multi(self, node, plan, targets):
        """Any number of targets: flood each component that touches target 0
        in turn and test it against every other target."""
        stones = self.stones(self.side(node.mover))
        ts = [self.em.const(t) for t in targets]
        dil_f = self._dilate(plan, "f")
        touch = " && ".join(f"lx::any(f & {t})" for t in ts[1:]) or "true"
        name = f"connected_multi_{self.em.fresh('k')}"
        self.em.helper(name, f"""    static __device__ __forceinline__ bool {name}(const BBW& mine) {{
        BBW rem = mine & {ts[0]};
        while (lx::any(rem)) {{
            BBW f = lx::onehot<W>(lx::select_bit(rem, 0));
            while (true) {{
                const BBW g = (f | {dil_f}) & mine;
                if (lx::equal(g, f)) break;
                f = g;
            }}
            if ({touch}) return true;
            rem = lx::andnot(rem, f);
        }}
        return false;
    }}""")
        return f"{name}({stones})"

    def _conn_update_code(self):
        """write_place tail: grow the placing side's reach sets.  One P1 slot
        and one P2 slot with the same direction plan share a single update
        on side-selected operands, so lanes of a warp with different movers
        do not diverge.  With a single update group the split form is also
        emitted (self.split_flood): write_place_pre leaves the flood's inputs
        in a Flood record, the rollout floods with the whole warp converged,
        and flood_post merges the result."""
        self.split_flood = None
        out = []
        by_side = {}
        for k, (sd, targets, plan) in enumerate(self.slot_info):
            by_side.setdefault(sd, []).append(k)
        merged = (len(self.slot_info) == 2 and sorted(by_side) == [0, 1]
                  and self.slot_info[0][2] == self.slot_info[1][2])
        groups = [(by_side[0][0], by_side[1][0])] if merged else [(k,) for k in
                                                                    range(len(self.slot_info))]
        for grp in groups:
            plan = self.slot_info[grp[0]][2]
            dil_f, dil_g = self._dilate(plan, "f"), self._dilate(plan, "g")
            dil_a = self._dilate(plan, "a")
            if len(grp) == 2:
                k0, k1 = grp
                c0 = self.em.const(self.slot_info[k0][1][0])
                c1 = self.em.const(self.slot_info[k1][1][0])
                head = (f"        {{\n            const bool s1 = side != 0;\n"
                        f"            BBW R = lx::sel(s1, {self._slot_get(k0)}, {self._slot_get(k1)});\n"
                        f"            const BBW t0 = lx::sel(s1, {c0}, {c1});")
                store = (f"if (s1) {{ {self._slot_set(k1, 'R')} }} else {{ {self._slot_set(k0, 'R')} }}")
                cond = "true"
            else:
                k = grp[0]
                sd = self.slot_info[k][0]
                head = (f"        {{\n            BBW R = {self._slot_get(k)};\n"
                        f"            const BBW t0 = {self.em.const(self.slot_info[k][1][0])};")
                store = self._slot_set(k, "R")
                cond = f"side == {sd}"
            dil_lw = self._dilate(plan, "x", ty="lx::LW<W>")
            flood = (f"                BBW g = (f | {dil_f}) & free_;\n"
                     f"                while (!lx::equal(g, f)) {{\n"
                     f"                    f = g;\n"
                     f"                    g = (f | {dil_f}) & free_;\n"
                     f"                }}")
            # grow inside the side's stones outside R; a converged full warp
            # floods cooperatively (lx::coop_flood), else each lane alone
            coop = (f"#if defined(__CUDA_ARCH__)\n"
                    f"            if (__activemask() == 0xffffffffu) {{\n"
                    f"                lx::coop_flood<W>(need, free_, f, [&](const lx::LW<W>& x) {{ return {dil_lw}; }});\n"
                    f"                solo = false;\n"
                    f"            }}\n"
                    f"#endif") if os.environ.get("LX_COOP_FLOOD", "1") != "0" else ""
            # the placed cell's plan neighbourhood and target-0 membership from
            # a per-cell table (one 16-byte load per ply instead of the
            # one-hot's four shifted copies)
            need_expr = f"({cond}) && lx::any((a & t0) | (({dil_a}) & R))"
            if os.environ.get("LX_NEIGHBOR_TABLE", "1") != "0":
                need_expr = self._need_table(plan, grp, cond)
            out.append(f"""{head}
            const BBW a = lx::onehot<W>(cell_bit(cell));
            const bool need = {need_expr};
            const BBW mine = side ? s.own1 : s.own0;
            const BBW free_ = lx::andnot(mine, R);
            BBW f = a;
            bool solo = true;
{coop}
            if (need) {{
                if (solo) {{
{flood}
                }}
                R = R | f;
                {store}
            }}
        }}""")
            # off by default: measured on the B200 (r2r/r2s,
            # profiles/r2r_ab_split_flood.jsonl) Hex 52.2 -> 47.2 G (its live
            # Flood record spills at 80 registers; at 128 registers it only
            # ties the fused ply), Yavalath +1.5 %
            if len(groups) == 1 and os.environ.get("LX_SPLIT_FLOOD", "0") != "0":
                pre = f"""{head}
            const BBW a = lx::onehot<W>(cell_bit(cell));
            fl.need = {need_expr};
            fl.free_ = lx::andnot(side ? s.own1 : s.own0, R);
            fl.f = a;
            fl.side = side;
        }}"""
                post = f"""        if (fl.need) {{
            const int side = fl.side;
{head.split(chr(10), 1)[1]}
            R = R | fl.f;
            {store}
        }}"""
                self.split_flood = (pre, post, dil_lw, dil_f)
        return "\n".join(out)

    def _need_table(self, plan, grp, cond):
        """`need` of a reach-set update from a constant per-cell table: words
        [0, W) = the cell's plan neighbours (as dilating {cell} gives them),
        word W = bit k set when the cell is in slot grp[k]'s target 0."""
        W = self.W
        name = f"NBT_{self.em.fresh('n')}"
        rows = []
        for c in range(self.C):
            b = int(self.bit_of[c])
            m = 0
            for d in plan:
                x = int(self.board.neighbors[d][c])
                if x != self.C:
                    m |= 1 << int(self.bit_of[x])
            flags = 0
            for k, slot in enumerate(grp):
                if bool(np.asarray(self.slot_info[slot][1][0])[c]):      # cell-indexed mask
                    flags |= 1 << k
            words = [(m >> (32 * i)) & 0xffffffff for i in range(W)] + [flags]
            rows.append("{" + ", ".join(f"0x{w:08x}u" for w in words) + "}")
        self.em.helper(name, f"    static __device__ __forceinline__ const u32* {name}(int c) {{\n"
                             f"        static __device__ const u32 t[{self.C}][{W + 1}] = {{\n            "
                             + ",\n            ".join(rows) + "};\n        return t[c];\n    }")
        loads = " | ".join(f"(__ldg({name}(cell) + {i}) & R.w[{i}])" for i in range(W))
        flag = ("((__ldg(" + name + f"(cell) + {W}) >> (s1 ? 1 : 0)) & 1u)" if len(grp) == 2
                else f"(__ldg({name}(cell) + {W}) & 1u)")
        return f"({cond}) && ({flag} || ({loads}) != 0u)"

    def _split_flood_code(self, owner, place_code, place_planes):
        """Game::SPLIT_FLOOD members (lx_rollout's converged flood): Flood,
        write_place_pre, flood_post and the lane-word dilation; stubs when
        the game has no single reach-set update."""
        sf = getattr(self, "split_flood", None)
        if sf is None or self.mech_kind != 0:
            return ("    static constexpr bool SPLIT_FLOOD = false;\n"
                    "    struct Flood { BBW free_, f; int need, side; };\n"
                    "    static __device__ __forceinline__ void write_place_pre(St& s, int cell, int mover, int phase, Flood& fl) "
                    "{ (void)s; (void)cell; (void)mover; (void)phase; fl.need = 0; }\n"
                    "    static __device__ __forceinline__ void flood_post(St&, const Flood&) {}\n"
                    "#if defined(__CUDA_ARCH__)\n"
                    "    static __device__ __forceinline__ lx::LW<W> flood_dil(const lx::LW<W>& x) { return x; }\n"
                    "#endif\n"
                    "    static __device__ __forceinline__ BBW flood_dil_bb(const BBW& f) { return f; }")
        pre, post, dil_lw, dil_f = sf
        return f"""    static constexpr bool SPLIT_FLOOD = true;
    struct Flood {{ BBW free_, f; int need, side; }};
    // write_place without the reach-set flood: its inputs go to fl
    static __device__ __forceinline__ void write_place_pre(St& s, int cell, int mover, int phase, Flood& fl) {{
        const int side = {owner};
{place_code}
        s.last_kind = 0; s.last_dest = cell; s.last_source = -1; s.last_mover = side;
        s.ldbp0 = side ? s.ldbp0 : cell;
        s.ldbp1 = side ? cell : s.ldbp1;
{place_planes}
{pre}
    }}
    // merge a flooded fl.f into the placing side's reach set
    static __device__ __forceinline__ void flood_post(St& s, const Flood& fl) {{
{post}
    }}
#if defined(__CUDA_ARCH__)
    static __device__ __forceinline__ lx::LW<W> flood_dil(const lx::LW<W>& x) {{ return {dil_lw}; }}
#endif
    static __device__ __forceinline__ BBW flood_dil_bb(const BBW& f) {{ return {dil_f}; }}"""

    def _conn_rebuild_code(self):
        """Reach sets from scratch (start position, lx_import)."""
        out = []
        for k, (sd, targets, plan) in enumerate(self.slot_info):
            t0 = self.em.const(targets[0])
            dil_f = self._dilate(plan, "f")
            out.append(f"""        {{
            const BBW mine = {"s.own1" if sd else "s.own0"};
            BBW f = mine & {t0};
            while (true) {{
                const BBW g = (f | {dil_f}) & mine;
                if (lx::equal(g, f)) break;
                f = g;
            }}
            {self._slot_set(k, "f")}
        }}""")
        return "\n".join(out)

    # -- functions / predicates -------------------------------------------

    def function(self, node):
        t = type(node)
        if t is n.ConstantFn:
            return str(int(node.value))
        if t is n.CountFn:
            return f"lx::popc({self.mask(node.mask)})"
        if t is n.ScoreFn:
            sd = self.side(node.who)
            return f"(({sd}) ? s.sc1 : s.sc0)"
        if t in (n.AddFn, n.MultiplyFn):
            op = " + " if t is n.AddFn else " * "
            return "(" + op.join(self.function(i) for i in node.items) + ")"
        if t is n.SubtractFn:
            return f"({self.function(node.a)} - {self.function(node.b)})"
        if t is n.LineFn:
            return self.line_count(node)
        if t is n.PatternFn:
            return self.pattern_count(node)
        if t is n.ConnectedFn:
            return f"(int){self.connected(node)}"
        _fail(f"function {t.__name__} is not lowered yet")

    def predicate(self, node, end_rule=False):
        t = type(node)
        if t in (n.PredAnd, n.PredOr):
            op = " && " if t is n.PredAnd else " || "
            return "(" + op.join(self.predicate(i, end_rule) for i in node.items) + ")"
        if t is n.PredNot:
            return f"(!{self.predicate(node.item, end_rule)})"
        if t is n.FunctionPred:
            if isinstance(node.fn, n.LineFn):
                return self.line_predicate(node.fn, end_rule)
            if isinstance(node.fn, n.ConnectedFn):
                return self.connected(node.fn)
            return f"({self.function(node.fn)} >= 1)"
        if t is n.ExistsPred:
            return f"lx::any({self.mask(node.mask)})"
        if t is n.FullBoardPred:
            return f"lx::equal(s.own0 | s.own1, {self.em.const(self.valid)})"
        if t is n.MoverIsPred:
            return f"(mover == {int(node.player)})"
        if t is n.EqualsPred:
            first = self.function(node.items[0])
            return "(" + " && ".join(f"({first} == {self.function(i)})"
                                     for i in node.items[1:]) + ")"
        if t in (n.GreaterEqPred, n.LessEqPred):
            op = ">=" if t is n.GreaterEqPred else "<="
            return f"({self.function(node.a)} {op} {self.function(node.b)})"
        if t is n.PassedPred:
            if node.who == n.BOTH:
                return "(s.pass_streak >= 2)"
            sd = self.side(node.who)
            return f"((({sd}) ? s.pf1 : s.pf0) != 0)"
        if t is n.LastMoveInPred:               # reference exprs.py:732-741
            m = self.mask(node.mask)
            return (f"(s.last_dest >= 0 && s.last_mover == mover && "
                    f"lx::test({m}, cell_bit(s.last_dest)))")
        if t is n.ActionWasPred:                # reference exprs.py:743-750
            sd = self.side(node.who)
            return f"(s.last_mover == ({sd}) && s.last_kind == {KIND_IDS[node.kind]})"
        if t is n.CanMoveAgainPred:             # reference exprs.py:752-757
            return f"can_move_again(s, mover, {KIND_IDS[node.kind]})"
        if t is n.NoLegalActionsPred:           # reference exprs.py:771-783
            if not end_rule:
                _fail("no_legal_actions outside an end condition")
            return "(next_count == 0)"
        _fail(f"predicate {t.__name__} is not lowered yet")

    def line_predicate(self, line, end_rule):
        """Global vs anchored line test, mirroring the reference's choice
        (compiler.py:122-135, 271-281; exprs.py:799-804).

        Where the reference anchors the test at last_dest, the global test is
        used when it is provably identical on every reachable state: the rule
        is a top-level `(if (line ...) <result>)`, stones are only added by
        the mover's own placements (no flips/promotion/movement; placement
        owner is the mover) and the start position holds no line -- then no
        non-terminal state ever contains a line, so any line after a move
        passes through the placed stone.  Otherwise the exact anchored form
        is emitted."""
        if end_rule and id(line) in self._anchored_lines:
            if self.use_probe and line.exclude is None and self.piece_mode == "single":
                return self.line_anchored_probe(line)   # exact anchored semantics, big boards
            if id(line) in self._global_ok:
                return self.line_exists(line)
            return self.line_anchored_exists(line)
        return self.line_exists(line)

    # ------------------------------------------------------------ rules

    def _decide_anchoring(self):
        self._anchored_lines = set()
        self._global_ok = set()
        start_has_line = self._start_boards()
        owners_mover = all(isinstance(p.mechanic, n.PlaceMechanic)
                           and p.mechanic.owner == n.MOVER for p in self.spec.phases)
        for line in self._anchor_candidates:
            own0, own1 = start_has_line
            if self._np_line(own0, line) or self._np_line(own1, line):
                continue      # reference keeps the global form (compiler.py:272-277)
            self.anchor_lines.add(line)
        if self._anchor_candidates and not self.anchor_lines and not self._last_action_base:
            self.layout["last_action"] = False
        for rule in self.spec.end_rules:
            for x in n.walk(rule.condition):
                if isinstance(x, n.FunctionPred) and isinstance(x.fn, n.LineFn) \
                        and x.fn in self.anchor_lines:
                    self._anchored_lines.add(id(x.fn))
                    top = rule.condition is x
                    if top and owners_mover and not self.has_flip:
                        self._global_ok.add(id(x.fn))

    def _np_line(self, owner_cells, line):
        """Start position holds a satisfied window for a side (reference
        _LineTables.satisfied, exprs.py:433-450: piece, exact, exclude)."""
        pid = self.piece_ids[line.piece]
        mine = owner_cells & (self._start_types == pid)
        excl = self._line_excluded(line) if line.exclude is not None else None
        nb = self.board.neighbors
        for d, cells in self.board.line_windows(line.length, line.orientation):
            if not all(mine[c] for c in cells):
                continue
            if excl is not None and excl[list(cells)].any():
                continue
            if line.exact:
                b = int(nb[OPPOSITE[d]][cells[0]])
                a = int(nb[d][cells[-1]])
                if (b != self.C and mine[b]) or (a != self.C and mine[a]):
                    continue
            return True
        return False

    def _start_boards(self):
        own = [np.zeros(self.C, dtype=bool), np.zeros(self.C, dtype=bool)]
        self._start_types = np.full(self.C, -1, dtype=np.int64)
        for sp in self.spec.start:
            cells = list(sp.cells) if sp.cells else \
                np.nonzero(self._static_union(sp.masks))[0].tolist()
            own[sp.player][cells] = True
            self._start_types[cells] = self.piece_ids[sp.piece]
        return own

    def lower(self):
        self._decide_anchoring()
        self._conn_tracking()
        NX = self.xbase + len(self.slot_info) * self.W
        spec = self.spec
        phases = spec.phases
        em = self.em
        # start position
        own = self._start_boards()
        start_scores = [0, 0]
        for sp in spec.start:
            cells = list(sp.cells) if sp.cells else \
                np.nonzero(self._static_union(sp.masks))[0].tolist()
            start_scores[sp.player] += len(cells)
        start_code = [f"        s.own0 = {em.const(own[0])};", f"        s.own1 = {em.const(own[1])};"]
        for t in range(1, self.NPL + 1):
            start_code.append(f"        {{ const BBW pl = {em.const(self._start_types == t)}; "
                              f"{self._plane_set(t, 'pl')} }}")
        if self.layout["scores"]:
            start_code.append(f"        s.sc0 = {start_scores[0]}; s.sc1 = {start_scores[1]};")

        # per-phase legality, write, effects
        legal_cases, fp_cases, eff_cases = [], [], []
        for pi, ph in enumerate(phases):
            mech = ph.mechanic
            if ph.force_pass:
                fp_cases.append(pi)
            if mech.effects:
                eff_cases.append(f"            case {pi}: {{\n{self.effects(mech.effects, mech)}\n"
                                 f"                break;\n            }}")
            if self.mech_kind != 0:
                continue
            dest = self.mask(mech.destination)
            legal = f"lx::andnot({em.const(self.valid)}, s.own0 | s.own1) & {dest}"
            if mech.result is not None:
                r = mech.result
                if (isinstance(r, n.ExistsPred) and isinstance(r.mask, n.CustodialMask)
                        and r.mask.mover == mech.owner):
                    legal += f" & {self.would_custodial(r.mask)}"
                else:
                    legal = self.result_sim(r, f"({legal})",
                                            "write_place(t, bit_cell(b), mover, t.phase);")
            legal_cases.append(f"            case {pi}: return {legal};")
        if self.mech_kind == 0:
            owner_side = [self.side(ph.mechanic.owner) for ph in phases]
            owner = owner_side[-1]
            if len(set(owner_side)) > 1:            # per-phase placement owners
                for pi in range(len(phases) - 2, -1, -1):
                    owner = f"(phase == {pi} ? {owner_side[pi]} : {owner})"
            place_planes = []
            for pi, ph in enumerate(phases):
                t = self.piece_ids[ph.mechanic.piece]
                if self.piece_mode == "planes" and t >= 1:
                    place_planes.append(f"        if (phase == {pi}) {{ BBW pl = {self._plane(t)}; "
                                        f"pl = pl | lx::onehot<W>(cell_bit(cell)); {self._plane_set(t, 'pl')} }}")
            place_planes = "\n".join(place_planes)
        elif self.mech_kind == 1:
            mech_code = self.movement_code(phases) + "\n" + self.movement_stubs()
        else:
            mech_code = self.gridworld_code(self.grid) + "\n" + self.movement_stubs()

        # end rules
        end_lines = []
        for rule in spec.end_rules:
            cond = self.predicate(rule.condition, end_rule=True)
            end_lines.append(f"        if ({cond}) return {self.result(rule.result)};")

        # advancement tables (reference compiler.py:251-267, 528-539)
        nph = len(phases)
        adv = []
        for pi, ph in enumerate(phases):
            order = list(ph.order)
            # turn_pos layout: keyed by the stored position; else the mover's
            # first position in the order (reference _pos_lookup)
            keys = (range(len(order)) if self.turn_pos else (0, 1))
            for key in keys:
                pos = key if self.turn_pos else (order.index(key) if key in order else 0)
                nxt = pos + 1
                wrap = nxt >= len(order)
                nphase = pi + 1 if (wrap and ph.kind == "once_through") else pi
                npos = 0 if wrap else nxt
                nplayer = phases[nphase].order[npos] if nphase < nph else 0
                cond = f"pos == {key}" if self.turn_pos else f"mover == {key}"
                adv.append(f"        if (phase == {pi} && {cond}) {{ np = {nplayer}; "
                           f"nphase = {nphase}; npos = {npos}; return; }}")
        conn = []
        for pi_, plan in enumerate(self.conn_plans):   # comp_labels[:, plan, :]
            dil = " | ".join(self.nb(d, "f") for d in plan)
            conn.append(f"""        {{
        short* lab = out + {pi_} * C;
        BBW done = lx::bb_zero<W>();
        for (int c = 0; c < C; c++) {{                    // ascending cell id = min label
            const int cb = cell_bit(c);
            const bool o0 = lx::test(s.own0, cb), o1 = lx::test(s.own1, cb);
            if (!o0 && !o1) {{ lab[c] = -1; continue; }}
            if (lx::test(done, cb)) continue;
            const BBW mine = lx::sel(o1, s.own0, s.own1);
            BBW f = lx::onehot<W>(cb);
            while (true) {{
                const BBW g = (f | {dil}) & mine;
                if (lx::equal(g, f)) break;
                f = g;
            }}
            done = done | f;
#pragma unroll
            for (int i = 0; i < W; i++) {{
                u32 bits = f.w[i];
                while (bits) {{
                    const int b = __ffs(bits) - 1;
                    lab[bit_cell(32 * i + b)] = (short)c;
                    bits &= bits - 1u;
                }}
            }}
        }}
        }}""")
        conn = "\n".join(conn)
        fp = " || ".join(f"phase == {p}" for p in fp_cases) or "false"
        conn_update = self._conn_update_code()
        conn_rebuild = self._conn_rebuild_code()
        self.ngc = {0: 1, 1: len(getattr(self, "groups", ())) or 1,
                    2: len(self.grid[2]) if self.grid else 1}[self.mech_kind]
        place_code = ("        lx::place_bit(s.own0, s.own1, cell_bit(cell), side);   // branchless\n"
                      "        if constexpr (ROW_MIRROR) { if (s.mirror_valid) rm_set(side, cell_bit(cell)); }")
        if self.mech_kind == 0:
            mech_code = f"""    static constexpr int MECH = 0;
    static __device__ __forceinline__ BBW legal(const St& s) {{
        const int mover = s.cur;
        const BBW me = mover ? s.own1 : s.own0;
        const BBW op = mover ? s.own0 : s.own1;
        (void)me; (void)op;
        switch (s.phase) {{
{chr(10).join(legal_cases)}
            default: return lx::bb_zero<W>();
        }}
    }}
    static __device__ __forceinline__ void write_place(St& s, int cell, int mover, int phase) {{
        const int side = {owner};
{place_code}
        s.last_kind = 0; s.last_dest = cell; s.last_source = -1; s.last_mover = side;
        s.ldbp0 = side ? s.ldbp0 : cell;
        s.ldbp1 = side ? cell : s.ldbp1;
{place_planes}
{conn_update}
    }}
{self.placement_stubs()}"""
            split_code = self._split_flood_code(owner, place_code, place_planes)
        else:
            split_code = self._split_flood_code(None, None, None)
        L = self.layout
        # rollout block shape: 256 threads; resident blocks per SM by board
        # size, from a B200 A/B at 2^22 envs over all 11 corpus games (same
        # stats; profiles/r1n_ab_minb_*.json): 4 on <= 16-cell boards (TTT
        # +2.3 %, gridworld +3.2 %), 3 up to 4 words (Wolf and Sheep +9.6 %,
        # Yavalath +8 %, draughts +3.7 %, Hex +2.3 %, C4/Reversi/DHS within
        # noise), 2 on the big boards (Pente -5.8 % at 3, Gomoku even)
        r_threads = 256
        r_minb = 4 if self.C <= 16 else (3 if self.W <= 4 else 2)
        r_threads = int(os.environ.get("LX_ROLLOUT_THREADS", r_threads))     # tuning overrides
        r_minb = int(os.environ.get("LX_ROLLOUT_MINB", r_minb))
        # batched game-over handling (lx_kernels.cuh): worth it for short games
        # only (measured on B200 at 2^22 envs, profiles/r1_tune_refill.jsonl:
        # TTT best 8-12, C4 best 6, Hex/Reversi/Pente best 1); board size bounds
        # the game length.  Env overrides for tuning.
        # (r2p/r2q re-tune with multi-ply passes: TTT 16 / 12 +6 % over 8 / 8;
        # C4, Hex, Reversi best as they were; profiles/r2p_ab_refill.jsonl)
        k_def = 8 if self.C <= 16 else (6 if self.C <= 48 else 1)
        w_def = k_def
        if self.C <= 16:
            k_def, w_def = 16, 12
        r_lanes = int(os.environ.get("LX_REFILL_LANES", str(k_def)))
        r_wait = int(os.environ.get("LX_REFILL_WAIT", str(w_def)))
        # plies per refill pass of lx_rollout: 2 on boards up to 128 cells (B200
        # A/B r2e, profiles/r2e_ab_select_unroll.jsonl: C4 +4.4 %, TTT +3.7 %,
        # Hex +1.4 %, Reversi +1.2 %), 1 beyond (Pente -11 %: its ply is large)
        # and for movement games (their doubled plies spill to the stack)
        # (r2j/r2k: 3 plies on <= 64 cells: TTT +9 %, C4 +1.3 %, Reversi +1.7 %
        # over 2; 4 is worse on TTT)
        r_unroll = int(os.environ.get("LX_PLY_UNROLL",
                                      ("3" if self.C <= 64 else "2")
                                      if self.C <= 128 and self.mech_kind == 0 else "1"))
        # funnel shifts as IMAD pairs on the FMA pipe: a win only where the
        # ALU pipe is saturated by shift-heavy Kogge-Stone fills (B200 A/B
        # r2g, profiles/r2g_ab_capture_stash_shiftfma.jsonl: Reversi +2.6 %;
        # C4 -2.5 %, Yavalath -4.3 %, Hex -1.2 %, Pente / TTT even)
        r_shift_fma = int(os.environ.get("LX_SHIFT_FMA", "1" if self.has_flip else "0"))
        src = f"""// generated by paper_2506_22609_b200.lowering for game "{spec.name}"
#define LX_BLOCK @@BLOCK@@
#define LX_ROLLOUT_THREADS @@RTHREADS@@
#define LX_ROLLOUT_MINB @@RMINB@@
#define LX_REFILL_LANES {r_lanes}
#define LX_REFILL_WAIT {r_wait}
#define LX_SELECT_SWAR {int(os.environ.get("LX_SELECT_SWAR", "1"))}
#define LX_PLY_UNROLL {r_unroll}
#define LX_SELECT_STASH {int(os.environ.get("LX_SELECT_STASH", "1"))}
#define LX_SHIFT_FMA {r_shift_fma}
#define LX_STATIC_CHUNKS {int(os.environ.get("LX_STATIC_CHUNKS", "1"))}
#define LX_ACQREL_TICKET {int(os.environ.get("LX_ACQREL_TICKET", "1"))}
#define LX_MASK_STREAM {int(os.environ.get("LX_MASK_STREAM", "1"))}
#define LX_CLUSTER_PUBLISH {int(os.environ.get("LX_CLUSTER_PUBLISH", "1"))}
#define LX_PUBLISH_INLINE @@PUBINL@@
#define LX_EARLY_DRAW @@EARLY@@
#define LX_STEP_MINB {int(os.environ.get("LX_STEP_MINB", "4"))}
#include "lx_core.cuh"

struct Game {{
    static constexpr int C = {self.C}, W = {self.W}, NX = {NX}, A = {self.A}, PASS = {self.PASS};
    static constexpr int FIRST_PLAYER = {phases[0].order[0]}, NPHASE = {nph};
    static constexpr bool L_SCORES = {str(L['scores']).lower()}, L_PASSING = {str(L['passing']).lower()};
    static constexpr bool L_LAST = {str(L['last_action']).lower()}, L_PHASE = {str(L['phase']).lower()};
    static constexpr bool L_TURNPOS = {str(L['turn_pos']).lower()};
    static constexpr bool IDENT = {str(self.ident).lower()};   // bit position == cell id
    static constexpr int NB = {self.NB};                       // bit slots (embedded grid)
    typedef lx::BB<W> BBW;
    static constexpr int NGC = {self.ngc};                     // cached move-group totals
    static constexpr int CONN_PLANS = {max(len(self.conn_plans), 1)};           // comp_labels planes
    static constexpr bool L_CONN = {str(bool(self.conn_plans)).lower()};
    typedef lx::State<W, NX, NGC> St;
{self._bitmap_code()}
@@CONSTS@@
@@RM@@
@@SPLIT@@
@@HELPERS@@
    static __device__ __forceinline__ void start(St& s) {{
{chr(10).join(start_code)}
        rebuild_ext(s);
    }}
    static __device__ __forceinline__ bool force_pass(int phase) {{ return {fp}; }}
    static constexpr int NT = {self.NT};                       // piece types
    static constexpr bool L_MUSTMOVE = {str(L['must_move']).lower()};
    static constexpr bool NEEDS_NEXT_COUNT = {str(self.needs_next_count).lower()};
{self._types_code()}
{self._transient_code()}
{mech_code}
    static __device__ __forceinline__ void effects(St& s, int cell, int mover, int phase) {{
        switch (phase) {{
{chr(10).join(eff_cases)}
            default: break;
        }}
    }}
    static __device__ __forceinline__ void advance(int phase, int pos, int mover, int& np,
                                                   int& nphase, int& npos) {{
        (void)pos; (void)mover;
{chr(10).join(adv)}
        np = 0; nphase = phase; npos = 0;
    }}
    static __device__ __forceinline__ int end_rules(const St& s, int mover, int next_count) {{
        const BBW me = mover ? s.own1 : s.own0;
        const BBW op = mover ? s.own0 : s.own1;
        (void)me; (void)op; (void)next_count;
{chr(10).join(end_lines)}
        return -1;
    }}
    static __device__ __forceinline__ void labels(const St& s, short* out) {{
{conn}
    }}
    static __device__ __forceinline__ void rebuild_ext(St& s) {{
{conn_rebuild}
    }}
}};

#include "lx_kernels.cuh"
"""
        nwords = state_words(self.W, NX, self.C, L, nph, self.mech_kind)
        src = src.replace("@@CONSTS@@", em.const_defs())
        src = src.replace("@@RM@@", self._rm_code())
        src = src.replace("@@SPLIT@@", split_code)
        # the row mirror (2 x (rows + 10) words per thread) fits 48 KB of static
        # shared memory per block at 128 threads, not 256: those games run
        # their per-env kernels and the rollout at 128 threads (4 rollout
        # blocks per SM keep 512 threads resident, as 2 x 256 before)
        if self.rm_used:
            r_threads = int(os.environ.get("LX_ROLLOUT_THREADS", 128))
            r_minb = int(os.environ.get("LX_ROLLOUT_MINB", 4))
        src = src.replace("@@BLOCK@@", "128" if self.rm_used else "256")
        # rollout epilogue inlined only where that register allocation wins
        # (row-mirror games; lx_kernels.cuh publish_stats)
        src = src.replace("@@PUBINL@@", os.environ.get("LX_PUBLISH_INLINE",
                                                       "1" if self.rm_used else "0"))
        # RNG chain ahead of the legality (lx_rules.cuh sample_action): B200
        # A/B r2zk at 2^22: Pente +2.3 %, C4 -0.4 %, TTT / Hex / Reversi within
        # noise, no latency gain at B=1024 -- on for the long row-mirror plies
        src = src.replace("@@EARLY@@", os.environ.get("LX_EARLY_DRAW",
                                                      "1" if self.rm_used else "0"))
        src = src.replace("@@RTHREADS@@", str(r_threads)).replace("@@RMINB@@", str(r_minb))
        src = src.replace("@@HELPERS@@", "\n".join(em.helpers.values()))
        info = {"name": spec.name, "C": self.C, "A": self.A, "W": self.W, "NX": NX,
                "pass_index": self.PASS, "layout": dict(self.layout),
                "nwords": nwords, "nq": (nwords + 3) // 4,
                "first_player": int(phases[0].order[0]), "nphase": nph,
                "observation_planes": 2 * self.NT + 1, "mechanics": self.mech_kind,
                "codec": {0: "placement", 1: "movement", 2: "gridworld"}[self.mech_kind],
                "grid_directions": list(self.grid[2]) if self.grid else [],
                "piece_mode": self.piece_mode, "piece_names": list(self.piece_ids)}
        return Lowered(name=spec.name, source=src, info=info)

    def effects(self, effs, mech):
        """Ordered effect list (reference effects.py:17-133), compiled in the
        anchored context (reference compiler.py:224-228)."""
        out = []
        self.anchored_ctx = True
        try:
            for e in effs:
                out.append(self.effect(e))
        finally:
            self.anchored_ctx = False
        return "\n".join(out)

    def effect(self, e):
        """One effect as a block that sees the board as left by the previous
        effects (me / op re-read).  Any effect but a mirrored capture may
        change the boards, so it invalidates the shared-memory mirror."""
        code = self._effect(e)
        ind = "                "
        if "capture_probe_" not in code and "capture_rm_" not in code:
            code += f"\n{ind}s.mirror_fresh = 0; s.mirror_valid = 0;"
        return (f"{ind}{{ const BBW me = mover ? s.own1 : s.own0; const BBW op = mover ? s.own0 : s.own1;\n"
                f"{ind}  (void)me; (void)op;\n{code}\n{ind}}}")

    def _effect(self, e):
        t = type(e)
        ind = "                "
        if t is n.FlipEffect:
            m = self.mask(e.mask)
            sd = self.side(e.mover)
            # branchless (lanes of a warp hold different movers)
            return (f"{ind}{{ const BBW cells = {m} & (s.own0 | s.own1); const bool fs = ({sd}) != 0;\n"
                    f"{ind}  s.own0 = lx::sel(fs, s.own0 | cells, lx::andnot(s.own0, cells));\n"
                    f"{ind}  s.own1 = lx::sel(fs, lx::andnot(s.own1, cells), s.own1 | cells); }}")
        if t is n.CaptureEffect:
            fast = self.capture_rm_block(e, ind)
            if fast is not None:
                return fast
            fast = self.capture_probe_block(e, ind)
            if fast is not None:
                return fast
            m = self.mask(e.mask)
            inc = ""
            if e.increment_score:
                inc = (f"\n{ind}  {{ const int g = lx::popc(cells); "
                       f"if (mover) s.sc1 += g; else s.sc0 += g; }}")
            mark = ""
            if self.transient:                  # effects.py:45-46
                mark = f"\n{ind}  {{ const BBW cm = {self._tplane(1)} | cells; {self._tplane_set(1, 'cm')} }}"
            return (f"{ind}{{ const BBW cells = {m} & (s.own0 | s.own1);{inc}{mark}\n"
                    + self._clear_cells_code("cells", ind + "  ") + f" }}")
        if t is n.PromoteEffect:                # reference effects.py:67-85
            m = self.mask(e.mask)
            sd = self.side(e.mover)
            fr, to = self.piece_ids[e.from_piece], self.piece_ids[e.to_piece]
            if self.piece_mode != "planes" and fr != to:
                _fail("promotion needs piece-type planes")
            lines = [f"{ind}{{ const BBW me = mover ? s.own1 : s.own0; const BBW op = mover ? s.own0 : s.own1;",
                     f"{ind}  (void)me; (void)op;",
                     f"{ind}  const BBW cells = {m} & {self.piece_bb(e.from_piece)} & {self.stones(self.side(e.mover)) if sd in ('mover', '(1 - mover)') else ('s.own1' if sd == '1' else 's.own0')};"]
            if fr >= 1:
                lines.append(f"{ind}  {{ const BBW pl = lx::andnot({self._plane(fr)}, cells); "
                             f"{self._plane_set(fr, 'pl')} }}")
            if to >= 1:
                lines.append(f"{ind}  {{ const BBW pl = {self._plane(to)} | cells; {self._plane_set(to, 'pl')} }}")
            if self.transient:                  # effects.py:83-84
                lines.append(f"{ind}  {{ const BBW pm = {self._tplane(2)} | cells; "
                             f"{self._tplane_set(2, 'pm')} }}")
            lines.append(f"{ind}}}")
            return "\n".join(lines)
        if t is n.ExtraTurnEffect:              # reference effects.py:104-115
            sd = self.side(e.who)
            return f"{ind}s.ovr = {sd};" + (" s.samep = 1;" if e.same_piece else "")
        if t in (n.SetScoreEffect, n.IncrementScoreEffect):
            sd = self.side(e.who)
            fn = self.function(e.fn)
            op = "=" if t is n.SetScoreEffect else "+="
            return (f"{ind}{{ const BBW me = mover ? s.own1 : s.own0; const BBW op = mover ? s.own0 : s.own1;\n"
                    f"{ind}  (void)me; (void)op; const int v = {fn};\n"
                    f"{ind}  if ({sd}) s.sc1 {op} v; else s.sc0 {op} v; }}")
        if t is n.ConditionalEffect:
            cond = self.predicate(e.condition)
            then = self.effect(e.then_effect)
            other = self.effect(e.else_effect) if e.else_effect is not None else ""
            return (f"{ind}{{ const BBW me = mover ? s.own1 : s.own0; const BBW op = mover ? s.own0 : s.own1;\n"
                    f"{ind}  (void)me; (void)op;\n"
                    f"{ind}  if ({cond}) {{\n{then}\n{ind}  }} else {{\n{other}\n{ind}  }} }}")
        _fail(f"effect {t.__name__} is not lowered yet")

    def result(self, res):
        """(reference compiler.py:582-597)"""
        if res.kind == "draw":
            return "0"
        if res.kind == "by_score":
            return "(s.sc0 > s.sc1 ? 1 : (s.sc1 > s.sc0 ? 2 : 0))"
        if res.who == n.BOTH:
            return "0"
        sd = self.side(res.who)
        if res.kind == "lose":
            return f"(1 + (1 - ({sd})))"
        return f"(1 + ({sd}))"


def state_words(W, NX, C, layout, nphase, mech):
    """32-bit words per env of the device state (mirror of lx::Layout in
    csrc/device/lx_rules.cuh): boards + private words, seed, int32 scores,
    then the packed meta bit fields the game keeps."""
    cb = int(C).bit_length()
    bits = 32 * (2 * W + NX + 2 + (2 if layout["scores"] else 0))
    bits += 32 + 1 + 1 + 1 + 2                       # move_count, cur, term, trunc, outcome
    bits += int(nphase).bit_length() if layout["phase"] else 0
    bits += 5 if layout["turn_pos"] else 0
    bits += 18 if layout["passing"] else 0           # pass_streak int16 + two flags
    if layout["last_action"]:
        bits += 2 + 3 + 3 * cb + (cb if mech != 0 else 0)
    bits += cb if layout["must_move"] else 0
    return (bits + 31) // 32


def lower_game(spec):
    try:
        return GameLowering(spec).lower()
    except KeyError as exc:
        raise CompileError("lower", str(exc)) from exc
