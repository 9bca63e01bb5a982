"""Lowering of movement and gridworld mechanics.

The reference keeps movement legality as per-source count matrices over
"move groups" -- one (move alternative, direction slot) pair each -- and
samples the r-th legal action in group order, then source-cell order, then
distance along the ray (reference mechanics.py:44-404).  Here each group
becomes a few whole-board bit operations on one env's bitboards:

  step   c = S & nb_d(E)                          (S: mover's pieces of the
  hop    c = S & nb_d(OV) & walk_d^2(E)            group's type, restricted to
  slide  R_k = R_{k-1} & walk_d^k(E),  R_0 = S     must_move; E: empty cells)

so a group's legal-action count is popc(c) (slides: sum_k popc(R_k)), the
r-th action of a step/hop group is the r-th set bit of c, and a slide picks
its source by walking the (few) source bits in ascending order.  Direction
slots whose P1 / P2 directions differ (forward_left, ...) select per mover.

Gridworld (reference mechanics.py:518-608) has one walker; its actions are
the board directions that lead to an empty cell.

Generated interface (consumed by csrc/device/lx_rules.cuh, MECH 1 / 2):
  count_moves(s, tot)          per-group totals after priority filtering
  select_move(s, r, tot, hint) r-th legal action; hint = its group
  move_legal(s, a)             first-claiming group exists and is active
  apply_move(s, a, mover, hint)
  enum_moves(s, f)             f(action) for every legal action (masks)
  can_move_again(s, mover, kind)
"""

from __future__ import annotations

from dataclasses import dataclass

from . import nodes as n
from .geometry import direction_pairs, resolve_direction

KIND_PLACE, KIND_STEP, KIND_HOP, KIND_SLIDE, KIND_PASS = 0, 1, 2, 3, 4   # state.py:23-31
KIND_IDS = {"place": KIND_PLACE, "step": KIND_STEP, "hop": KIND_HOP, "slide": KIND_SLIDE,
            "pass": KIND_PASS}
BIG_PRIO = 10 ** 6                                                     # mechanics.py:22


@dataclass
class MoveGroup:
    """One (move alternative, direction slot) -- reference MoveGroup
    (mechanics.py:44-82)."""
    kind: int
    piece: str
    prio: int
    d1: str
    d2: str
    over_piece: str = ""
    hop_over: str = ""
    capture: bool = False
    L: int = 1
    phase: int = 0
    legal: str = ""          # placement pseudo-group: legal-cell bitboard expression
    owner: str = ""          # placement pseudo-group: owner side expression

    @property
    def symmetric(self):
        return self.d1 == self.d2


class MoveLoweringMixin:
    """Methods of GameLowering for MoveMechanic / gridworld phases."""

    # ------------------------------------------------------------ analysis

    def _movement_groups(self, mech):
        """reference compiler.py:311-327 (group order = move order x slot order)."""
        groups = []
        for mv in mech.moves:
            pairs = direction_pairs(mv.directions or ("any",), self.forward, self.board)
            for d1, d2 in pairs:
                if isinstance(mv, n.StepMove):
                    groups.append(MoveGroup(KIND_STEP, mv.piece, mv.priority, d1, d2))
                elif isinstance(mv, n.HopMove):
                    groups.append(MoveGroup(KIND_HOP, mv.piece, mv.priority, d1, d2,
                                            over_piece=mv.over_piece, hop_over=mv.hop_over,
                                            capture=bool(mv.capture)))
                elif isinstance(mv, n.SlideMove):
                    L = max(max(self.board.ray_length(d1), 1), max(self.board.ray_length(d2), 1))
                    if mv.distance:
                        L = min(L, mv.distance)
                    groups.append(MoveGroup(KIND_SLIDE, mv.piece, mv.priority, d1, d2, L=L))
                else:
                    self._fail_move(f"move {type(mv).__name__}")
        return groups

    @staticmethod
    def _fail_move(msg):
        from .lowering import _fail
        _fail(f"{msg} is not lowered yet")

    def _detect_gridworld(self):
        """reference compiler.py:155-183: single mover, step-only moves of one
        piece, no capture/flip, exactly one start cell for that player."""
        spec = self.spec
        players = {p for ph in spec.phases for p in ph.order}
        if len(players) != 1:
            return None
        player = next(iter(players))
        dirs, piece = [], None
        for ph in spec.phases:
            mech = ph.mechanic
            if not isinstance(mech, n.MoveMechanic):
                return None
            for mv in mech.moves:
                if not isinstance(mv, n.StepMove):
                    return None
                if piece is not None and mv.piece != piece:
                    return None
                piece = mv.piece
                dirs.extend(resolve_direction(mv.directions or ("any",), player,
                                              self.forward, self.board))
        for x in n.walk(spec):
            if isinstance(x, (n.CaptureEffect, n.FlipEffect)):
                return None
        start_cells = 0
        for sp in spec.start:
            if sp.player == player:
                start_cells += len(sp.cells) if sp.cells else int(self._static_union(sp.masks).sum())
        if start_cells != 1:
            return None
        ordered = tuple(d for d in self.board.directions if d in dirs)
        return player, piece, ordered

    def _group_claim_safe(self, groups):
        """safe[g]: no earlier group can claim an action group g generates, so
        the sampled group is the claiming group (reference apply claims the
        first matching group in order, mechanics.py:283-322).  Geometric
        overlap test per mover; a hop and a slide along the same direction are
        exclusive (the jumped cell is occupied vs empty)."""
        C = self.C
        nbr = self.board.neighbors

        def dests(g, d, src):
            nt = nbr[d]
            if g.kind == KIND_STEP:
                x = int(nt[src])
                return {x} if x != C else set()
            if g.kind == KIND_HOP:
                x = int(nt[src])
                x = int(nt[x]) if x != C else C
                return {x} if x != C else set()
            out, x = set(), src
            for _ in range(g.L):
                x = int(nt[x]) if x != C else C
                if x == C:
                    break
                out.add(x)
            return out

        safe = []
        for gi, g in enumerate(groups):
            ok = True
            for h in groups[:gi]:
                if h.piece != g.piece:
                    continue
                for mover in (0, 1):
                    dg = g.d1 if mover == 0 else g.d2
                    dh = h.d1 if mover == 0 else h.d2
                    if {g.kind, h.kind} == {KIND_HOP, KIND_SLIDE} and dg == dh:
                        continue
                    for src in range(C):
                        if dests(g, dg, src) & dests(h, dh, src):
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            safe.append(ok)
        return safe

    # ------------------------------------------------------------ piece types

    def _setup_piece_types(self):
        """Piece-type representation on the device.

        single    one type: board_piece is 0 wherever a stone is
        by_owner  two types, each owned by one player (Wolf and Sheep): the
                  owner determines the type, no planes needed
        planes    one extra bitboard per type >= 1 (type 0 = occupied cells in
                  no plane), stored in the rule-private words"""
        pieces = list(self.spec.equipment.pieces)
        self.NT = len(pieces)
        types = {type(x) for x in n.walk(self.spec)}
        self.type_owner = None
        if self.NT == 1:
            self.piece_mode = "single"
        else:
            owners = [p.owner for p in pieces]
            mode = "planes"
            if (self.NT == 2 and sorted(str(o) for o in owners) == ["0", "1"]
                    and n.PromoteEffect not in types and n.FlipEffect not in types):
                consistent = all(sp.player == owners[self.piece_ids[sp.piece]]
                                 for sp in self.spec.start)
                for ph in self.spec.phases:
                    m = ph.mechanic
                    if isinstance(m, n.PlaceMechanic):
                        consistent = False          # placement owner is resolved per mover
                if consistent:
                    mode = "by_owner"
                    self.type_owner = [int(o) for o in owners]
            self.piece_mode = mode
        self.NPL = (self.NT - 1) if self.piece_mode == "planes" else 0
        self.xbase = self.NPL * self.W

    def _plane(self, t):
        W = self.W
        words = ", ".join(f"s.ext[{(t - 1) * W + i}]" for i in range(W))
        return f"BBW{{{{{words}}}}}"

    def _plane_set(self, t, var):
        W = self.W
        return " ".join(f"s.ext[{(t - 1) * W + i}] = {var}.w[{i}];" for i in range(W))

    def piece_bb(self, name):
        """Expression: cells holding a piece of type `name` (any owner)."""
        t = self.piece_ids[name]
        if self.piece_mode == "single":
            return "(s.own0 | s.own1)"
        if self.piece_mode == "by_owner":
            return "s.own1" if self.type_owner[t] else "s.own0"
        if t >= 1:
            return self._plane(t)
        others = " | ".join(self._plane(k) for k in range(1, self.NT))
        return f"lx::andnot(s.own0 | s.own1, {others})"

    def piece_filter(self, name, expr):
        """expr restricted to pieces of type `name` (no-op with one type)."""
        if self.piece_mode == "single":
            return expr
        return f"({expr} & {self.piece_bb(name)})"

    def _types_code(self):
        """type_bb / piece_at / set_piece / clear_types (export, import,
        observation; reference board_piece semantics)."""
        NT = self.NT
        cases = "\n".join(f"            case {t}: return {self.piece_bb(p.name)};"
                          for t, p in enumerate(self.spec.equipment.pieces))
        type_bb = (f"    static __device__ __forceinline__ BBW type_bb(const St& s, int t) {{\n"
                   f"        switch (t) {{\n{cases}\n            default: return lx::bb_zero<W>();\n"
                   f"        }}\n    }}")
        if self.piece_mode == "single":
            at = "        return 0;"
            setp = "        (void)s; (void)b; (void)t;"
            clr = "        (void)s;"
        elif self.piece_mode == "by_owner":
            at = f"        return lx::test(s.own0, b) ? {self.type_owner.index(0)} : {self.type_owner.index(1)};"
            setp = "        (void)s; (void)b; (void)t;"
            clr = "        (void)s;"
        else:
            at = "\n".join(f"        if (lx::test({self._plane(t)}, b)) return {t};"
                           for t in range(1, NT)) + "\n        return 0;"
            setp = "\n".join(f"        if (t == {t}) s.ext[{(t - 1) * self.W} + (b >> 5)] |= 1u << (b & 31);"
                             for t in range(1, NT))
            clr = "\n".join(f"        s.ext[{i}] = 0u;" for i in range(self.NPL * self.W))
        return (f"{type_bb}\n"
                f"    static __device__ __forceinline__ int piece_at(const St& s, int b) {{\n{at}\n    }}\n"
                f"    static __device__ __forceinline__ void set_piece(St& s, int b, int t) {{\n{setp}\n    }}\n"
                f"    static __device__ __forceinline__ void clear_types(St& s) {{\n{clr}\n    }}")

    def _tplane(self, k):
        """Transient mask k (0 hopped, 1 captured, 2 promoted) as a BBW."""
        W, T = self.W, self.tbase
        words = ", ".join(f"s.ext[{T + k * W + i}]" for i in range(W))
        return f"BBW{{{{{words}}}}}"

    def _tplane_set(self, k, var):
        W, T = self.W, self.tbase
        return " ".join(f"s.ext[{T + k * W + i}] = {var}.w[{i}];" for i in range(W))

    def _transient_code(self):
        """clear_transient (start of every ply, compiler.py:473-476) and the
        (B, C) bool export / import of the three transient masks."""
        if not self.transient:
            return ("    static __device__ __forceinline__ void clear_transient(St&) {}\n"
                    "    static __device__ __forceinline__ void export_transient(const St&, "
                    "unsigned char*, unsigned char*, unsigned char*) {}\n"
                    "    static __device__ __forceinline__ void import_transient(St&, "
                    "const unsigned char*, const unsigned char*, const unsigned char*) {}")
        W, T = self.W, self.tbase
        clr = " ".join(f"s.ext[{T + i}] = 0u;" for i in range(3 * W))
        return f"""    static __device__ __forceinline__ void clear_transient(St& s) {{ {clr} }}
    static __device__ __forceinline__ void export_transient(const St& s, unsigned char* h,
                                                            unsigned char* c, unsigned char* p) {{
        const BBW hb = {self._tplane(0)}, cb = {self._tplane(1)}, pb = {self._tplane(2)};
        for (int x = 0; x < C; x++) {{
            const int b = cell_bit(x);
            h[x] = lx::test(hb, b); c[x] = lx::test(cb, b); p[x] = lx::test(pb, b);
        }}
    }}
    static __device__ __forceinline__ void import_transient(St& s, const unsigned char* h,
                                                            const unsigned char* c,
                                                            const unsigned char* p) {{
        BBW hb = lx::bb_zero<W>(), cb = lx::bb_zero<W>(), pb = lx::bb_zero<W>();
        for (int x = 0; x < C; x++) {{
            const int b = cell_bit(x);
            if (h[x]) lx::setbit(hb, b);
            if (c[x]) lx::setbit(cb, b);
            if (p[x]) lx::setbit(pb, b);
        }}
        {self._tplane_set(0, 'hb')} {self._tplane_set(1, 'cb')} {self._tplane_set(2, 'pb')}
    }}"""

    def _clear_cells_code(self, cells, ind):
        """Remove whatever stands on `cells` (both owners, every type plane)."""
        out = [f"{ind}s.own0 = lx::andnot(s.own0, {cells}); s.own1 = lx::andnot(s.own1, {cells});"]
        for t in range(1, self.NPL + 1):
            out.append(f"{ind}{{ const BBW pl = lx::andnot({self._plane(t)}, {cells}); "
                       f"{self._plane_set(t, 'pl')} }}")
        return "\n".join(out)

    # ------------------------------------------------------------ movement code

    def _shift_of(self, d):
        return self._shift[d]

    def _mv_prelude(self, mover="s.cur"):
        lines = [f"        const int mover = {mover};",
                 "        const BBW me = mover ? s.own1 : s.own0;",
                 "        const BBW op = mover ? s.own0 : s.own1;",
                 "        const BBW E = lx::andnot(" + self.em.const(self.valid) + ", s.own0 | s.own1);",
                 "        (void)me; (void)op; (void)E;"]
        if self.layout["must_move"]:
            lines.append(f"        const BBW MM = s.must_move >= 0 ? lx::onehot<W>(cell_bit(s.must_move)) "
                         f": {self.em.const(self.valid)};")
        return lines

    def _src_expr(self, g, must=True):
        e = self.piece_filter(g.piece, "me")
        if must and self.layout["must_move"]:
            e = f"({e} & MM)"
        return e

    def _over_expr(self, g):
        """Cells a hop may jump: occupied, of hop_over's side / over_piece
        (reference mechanics.py:149-167)."""
        e = "(s.own0 | s.own1)"
        if g.hop_over != "":
            e = self.stones(self.side(g.hop_over))
        if g.over_piece:
            e = f"({e} & {self.piece_bb(g.over_piece)})"
        return e

    def _count_plane(self, g, d, S):
        """Expression of the per-source legal bitboard of a step / hop group
        along direction d (sources S)."""
        if g.kind == KIND_STEP:
            return f"({S} & {self.nb(d, 'E')})"
        ov = self._over_expr(g)
        return f"({S} & {self.nb(d, ov)} & {self.walk(d, 2, 'E')})"

    def _slide_lines(self, g, d, S, per_k, ind):
        """Reach planes R_k of a slide group along d; per_k(k, var) emits the
        use of each plane."""
        out = [f"{ind}BBW R = {S};"]
        for k in range(1, g.L + 1):
            out.append(f"{ind}R = R & {self.walk(d, k, 'E')};")
            out += per_k(k, "R")
        return out

    def _group_count_code(self, gi, g, ind):
        """tot[gi] = number of legal actions of group g."""
        S = self._src_expr(g)
        if g.kind in (KIND_STEP, KIND_HOP):
            if g.symmetric:
                return [f"{ind}tot[{gi}] = lx::popc({self._count_plane(g, g.d1, S)});"]
            return [f"{ind}tot[{gi}] = lx::popc(lx::sel(mover != 0, {self._count_plane(g, g.d1, S)}, "
                    f"{self._count_plane(g, g.d2, S)}));"]
        out = []

        def body(d):
            lines = [f"{ind}{{", f"{ind}    int k_ = 0;"]
            lines += self._slide_lines(g, d, S, lambda k, v: [f"{ind}    k_ += lx::popc({v});"],
                                       ind + "    ")
            lines += [f"{ind}    tot[{gi}] = k_;", f"{ind}}}"]
            return lines
        if g.symmetric:
            out += body(g.d1)
        else:
            out.append(f"{ind}if (mover == 0) {{")
            out += body(g.d1)
            out.append(f"{ind}}} else {{")
            out += body(g.d2)
            out.append(f"{ind}}}")
        return out

    def _pick_helper(self, gi, g):
        """pick_g(s, r): r-th action of group g (reference mechanics.py:211-232)."""
        C = self.C
        name = f"pick_g{gi}"
        lines = self._mv_prelude()

        def one(d):
            Sd = self._shift_of(d)
            S = self._src_expr(g)
            if g.kind in (KIND_STEP, KIND_HOP):
                off = Sd if g.kind == KIND_STEP else 2 * Sd
                return [f"        {{ const BBW c = {self._count_plane(g, d, S)};",
                        "          const int x = lx::select_bit(c, r);",
                        f"          return bit_cell(x) * {C} + bit_cell(x + {off}); }}"]
            L = g.L
            out = ["        {", f"        BBW RK[{L}];"]
            out += self._slide_lines(g, d, S, lambda k, v: [f"        RK[{k - 1}] = {v};"], "        ")
            out += ["        BBW rem = RK[0];",
                    "        while (true) {",
                    "            const int x = lx::select_bit(rem, 0);",
                    "            int cnt = 0;",
                    "#pragma unroll",
                    f"            for (int k = 0; k < {L}; k++) cnt += lx::test(RK[k], x);",
                    f"            if (r < cnt) return bit_cell(x) * {C} + bit_cell(x + (r + 1) * {Sd});",
                    "            r -= cnt;",
                    "            lx::clearbit(rem, x);",
                    "        }",
                    "        }"]
            return out
        if g.symmetric:
            lines += one(g.d1)
        else:
            lines.append("        if (mover == 0) {")
            lines += one(g.d1)
            lines.append("        } else {")
            lines += one(g.d2)
            lines.append("        }")
        lines.append("        return -1;")
        body = "\n".join(lines)
        self.em.helper(name, f"    static __device__ __forceinline__ int {name}(const St& s, int r) {{\n"
                             f"{body}\n    }}")
        return name

    def _select_code(self, items):
        """Candidate planes of one phase's groups and the chosen action, given
        `g` (chosen group) and `rr` (index inside it) -- the r-th action over
        groups in order, then source cell, then distance (reference
        mechanics.py:199-232), without per-group branches: lanes of a warp pick
        different groups, so every group's candidate plane is built and the
        chosen one kept by select (divergent per-group code was the dominant
        cost).  Step / hop: r-th set bit of the chosen plane.  Slides: the
        reach planes R_1 >= .. >= R_L of each slide group become bit-sliced
        per-source counts and lx::select_weighted finds (source, distance) by
        prefix popcounts.  Placement: r-th legal cell."""
        C = self.C
        out = []
        pl = [(gi, g) for gi, g in items if g.kind == KIND_PLACE]
        sh = [(gi, g) for gi, g in items if g.kind in (KIND_STEP, KIND_HOP)]
        sl = [(gi, g) for gi, g in items if g.kind == KIND_SLIDE]
        for gi, g in pl:
            out.append(f"        if (g == {gi}) return bit_cell(lx::select_bit({g.legal}, rr));")

        def off_expr(g):
            k = 1 if g.kind == KIND_STEP else 2
            o1, o2 = k * self._shift_of(g.d1), k * self._shift_of(g.d2)
            return str(o1) if o1 == o2 else f"(mover ? {o2} : {o1})"
        if sh:
            out.append("        BBW cs = lx::bb_zero<W>();")
            out.append("        int off = 0;")
            for gi, g in sh:
                S = self._src_expr(g)
                if g.symmetric:
                    plane = self._count_plane(g, g.d1, S)
                else:
                    plane = (f"lx::sel(mover != 0, {self._count_plane(g, g.d1, S)}, "
                             f"{self._count_plane(g, g.d2, S)})")
                out.append(f"        {{ const BBW c = {plane}; "
                           f"cs = lx::sel(g == {gi}, cs, c); off = g == {gi} ? {off_expr(g)} : off; }}")
        if sl:
            NB = max(g.L for _, g in sl).bit_length()
            out.append(f"        BBW dg[{NB}];")
            out.append("#pragma unroll")
            out.append(f"        for (int j = 0; j < {NB}; j++) dg[j] = lx::bb_zero<W>();")
            out.append("        int ss = 0;")

            def digits(g, d, S, tag):
                lines = [f"            BBW R0_{tag} = {S};"]
                prev = f"R0_{tag}"
                for k in range(1, g.L + 1):
                    lines.append(f"            const BBW R{k}_{tag} = {prev} & {self.walk(d, k, 'E')};")
                    prev = f"R{k}_{tag}"
                for m in range(1, g.L + 1):
                    seg = f"R{m}_{tag}" if m == g.L else f"lx::andnot(R{m}_{tag}, R{m + 1}_{tag})"
                    lines.append(f"            const BBW G{m}_{tag} = {seg};")
                dig = []
                for j in range(NB):
                    parts = [f"G{m}_{tag}" for m in range(1, g.L + 1) if (m >> j) & 1]
                    dig.append(" | ".join(parts) if parts else "lx::bb_zero<W>()")
                return lines, dig
            for gi, g in sl:
                S = self._src_expr(g)
                out.append("        {")
                if g.symmetric:
                    lines, dig = digits(g, g.d1, S, "a")
                    out += lines
                    for j in range(NB):
                        out.append(f"            dg[{j}] = lx::sel(g == {gi}, dg[{j}], BBW({dig[j]}));")
                    out.append(f"            ss = g == {gi} ? {self._shift_of(g.d1)} : ss;")
                else:
                    la, da = digits(g, g.d1, S, "a")
                    lb, db = digits(g, g.d2, S, "b")
                    out += la + lb
                    for j in range(NB):
                        out.append(f"            dg[{j}] = lx::sel(g == {gi}, dg[{j}], "
                                   f"lx::sel(mover != 0, BBW({da[j]}), BBW({db[j]})));")
                    out.append(f"            ss = g == {gi} ? (mover ? {self._shift_of(g.d2)} : "
                               f"{self._shift_of(g.d1)}) : ss;")
                out.append("        }")
            cond = " || ".join(f"g == {gi}" for gi, _ in sl)
            out.append(f"        if ({cond}) {{")
            out.append("            int rem;")
            out.append(f"            const int x = lx::select_weighted<W, {NB}>(dg, rr, rem);")
            out.append(f"            return bit_cell(x) * {C} + bit_cell(x + (rem + 1) * ss);")
            out.append("        }")
        if sh:
            out.append("        const int x = lx::select_bit(cs, rr);")
            out.append(f"        return bit_cell(x) * {C} + bit_cell(x + off);")
        else:
            out.append("        return -1;")
        return "\n".join(out)

    def _match_helper(self, gi, g):
        """match_g(s, bs, bd): group g moves the piece on bit bs to bit bd
        (reference mechanics.py:287-318, without the source test)."""
        name = f"match_g{gi}"
        lines = self._mv_prelude()

        def one(d):
            Sd = self._shift_of(d)
            k1 = self.em.const(self._walk_ok(d, 1))
            if g.kind == KIND_STEP:
                return [f"        return lx::test({k1}, bs) && bd == bs + {Sd} && lx::test(E, bd);"]
            if g.kind == KIND_HOP:
                k2 = self.em.const(self._walk_ok(d, 2))
                return [f"        return lx::test({k2}, bs) && bd == bs + {2 * Sd} && "
                        f"lx::test({self._over_expr(g)}, bs + {Sd}) && lx::test(E, bd);"]
            out = ["        bool clear = true, arrived = false;"]
            for k in range(1, g.L + 1):
                kk = self.em.const(self._walk_ok(d, k))
                out.append(f"        clear = clear && lx::test({kk}, bs) && lx::test(E, bs + {k * Sd});")
                out.append(f"        arrived = arrived || (clear && bd == bs + {k * Sd});")
            out.append("        return arrived;")
            return out
        if g.symmetric:
            lines += one(g.d1)
        else:
            lines.append("        if (mover == 0) {")
            lines += one(g.d1)
            lines.append("        } else {")
            lines += one(g.d2)
            lines.append("        }")
        body = "\n".join(lines)
        self.em.helper(name, f"    static __device__ __forceinline__ bool {name}(const St& s, int bs, int bd) {{\n"
                             f"{body}\n    }}")
        return name

    def _enum_code(self, gi, g):
        """f(action) for each legal action of group g."""
        C = self.C

        def bits(var, off):
            return [f"#pragma unroll",
                    f"            for (int w_ = 0; w_ < W; w_++) {{",
                    f"                u32 b_ = {var}.w[w_];",
                    f"                while (b_) {{",
                    f"                    const int x = 32 * w_ + __ffs(b_) - 1;",
                    f"                    b_ &= b_ - 1u;",
                    f"                    f(bit_cell(x) * {C} + bit_cell(x + {off}));",
                    f"                }}",
                    f"            }}"]

        def one(d):
            Sd = self._shift_of(d)
            S = self._src_expr(g)
            if g.kind in (KIND_STEP, KIND_HOP):
                off = Sd if g.kind == KIND_STEP else 2 * Sd
                return [f"            {{ const BBW c = {self._count_plane(g, d, S)};"] + bits("c", off) + ["            }"]
            out = ["            {"]
            out += self._slide_lines(g, d, S, lambda k, v: ["            {"] + bits(v, k * Sd) + ["            }"],
                                     "            ")
            out.append("            }")
            return out
        out = [f"        if (tot[{gi}] > 0) {{"]
        if g.symmetric:
            out += one(g.d1)
        else:
            out.append("        if (mover == 0) {")
            out += one(g.d1)
            out.append("        } else {")
            out += one(g.d2)
            out.append("        }")
        out.append("        }")
        return out

    def _place_group(self, pi, mech):
        """A placement phase inside a movement-codec game: one pseudo-group
        whose actions are the legal cells (reference PlacementMechanics,
        mechanics.py:415-515)."""
        from .lowering import _fail
        g = MoveGroup(KIND_PLACE, mech.piece, 0, "", "", phase=pi, owner=self.side(mech.owner))
        wname = f"place_write_p{pi}"
        self.em.helper(wname, f"""    static __device__ __forceinline__ void {wname}(St& s, int a, int mover) {{
{self._place_write(g, "        ")}
    }}""")
        legal = f"(lx::andnot({self.em.const(self.valid)}, s.own0 | s.own1) & {self.mask(mech.destination)})"
        if mech.result is not None:
            r = mech.result
            if (isinstance(r, n.ExistsPred) and isinstance(r.mask, n.CustodialMask)
                    and r.mask.mover == mech.owner):
                legal = f"({legal} & {self.would_custodial(r.mask)})"
            else:
                legal = self.result_sim(r, legal, f"{wname}(t, bit_cell(b), mover);")
        g.legal = legal
        return g

    def _place_write(self, g, ind):
        """_write_placement (mechanics.py:463-479) of a placement phase."""
        t = self.piece_ids[g.piece]
        plane = ""
        if self.piece_mode == "planes" and t >= 1:
            plane = f"\n{ind}{{ BBW pl = {self._plane(t)} | oh; {self._plane_set(t, 'pl')} }}"
        return (f"{ind}const int side = {g.owner};\n"
                f"{ind}const BBW oh = lx::onehot<W>(cell_bit(a));\n"
                f"{ind}s.own0 = lx::sel(side != 0, s.own0 | oh, s.own0);\n"
                f"{ind}s.own1 = lx::sel(side != 0, s.own1, s.own1 | oh);{plane}\n"
                f"{ind}s.last_kind = {KIND_PLACE}; s.last_source = -1; s.last_dest = a; "
                f"s.last_mover = side;\n"
                f"{ind}s.ldbp0 = side ? s.ldbp0 : a;\n"
                f"{ind}s.ldbp1 = side ? a : s.ldbp1;")

    def movement_code(self, phases):
        """struct Game members of a movement-codec game (MECH 1): every phase
        is a set of move groups (or one placement pseudo-group), dispatched on
        the state's phase; the dead phase after a finished once_through
        sequence has no legal action (compiler.py:251-267, 379-392)."""
        from .lowering import _fail
        groups, by_phase = [], []
        for pi, ph in enumerate(phases):
            mech = ph.mechanic
            if isinstance(mech, n.MoveMechanic):
                gs = self._movement_groups(mech)
                if not gs:
                    _fail("movement phase without moves")
                for g in gs:
                    g.phase = pi
            else:
                gs = [self._place_group(pi, mech)]
            by_phase.append(list(range(len(groups), len(groups) + len(gs))))
            groups += gs
        self.groups = groups
        NG = len(groups)
        C = self.C
        prios = [g.prio for g in groups]
        multi = len({g.prio for g in groups if g.kind != KIND_PLACE}) > 1
        safe = [True] * NG
        for idx in by_phase:
            mv = [i for i in idx if groups[i].kind != KIND_PLACE]
            for i, ok in zip(mv, self._group_claim_safe([groups[i] for i in mv])):
                safe[i] = ok
        pre = "\n".join(self._mv_prelude())
        is_place = {pi: groups[idx[0]].kind == KIND_PLACE for pi, idx in enumerate(by_phase)}

        def phase_switch(body_of, default="break;"):
            out = ["        switch (s.phase) {"]
            for pi, idx in enumerate(by_phase):
                body = body_of(pi, idx)
                if body is None:
                    continue
                out.append(f"            case {pi}: {{")
                out.append(body)
                out.append("            } break;")
            out.append(f"            default: {default}")
            out.append("        }")
            return "\n".join(out)

        # counts (+ priority activity, reference mechanics.py:188-197)
        def count_body(pi, idx):
            lines = []
            for gi in idx:
                g = groups[gi]
                if g.kind == KIND_PLACE:
                    lines.append(f"        tot[{gi}] = lx::popc({g.legal});")
                else:
                    lines += self._group_count_code(gi, g, "        ")
            return "\n".join(lines)
        zero = " ".join(f"tot[{gi}] = 0;" for gi in range(NG))
        raw = f"        {zero}\n" + phase_switch(count_body)
        filt = []
        if multi:
            filt.append(f"        int minp = {BIG_PRIO};")
            for gi, g in enumerate(groups):
                filt.append(f"        if (tot[{gi}] > 0 && {g.prio} < minp) minp = {g.prio};")
            for gi, g in enumerate(groups):
                filt.append(f"        if ({g.prio} != minp) tot[{gi}] = 0;")
        filt.append("        int n_ = 0;")
        for gi in range(NG):
            filt.append(f"        n_ += tot[{gi}];")
        filt = "\n".join(filt)
        scan = ["        int g = -1, rr = r;"]
        for gi in range(NG):
            scan.append(f"        {{ const bool h = g < 0 && rr < tot[{gi}]; "
                        f"rr = (g < 0 && !h) ? rr - tot[{gi}] : rr; g = h ? {gi} : g; }}")
        scan.append("        hint = g;")
        scan.append("        if (g < 0) return -1;")
        sel = "\n".join(scan) + "\n" + phase_switch(
            lambda pi, idx: self._select_code([(gi, groups[gi]) for gi in idx]))
        matches = {gi: self._match_helper(gi, g) for gi, g in enumerate(groups)
                   if g.kind != KIND_PLACE}

        def claim_body(pi, idx):
            if is_place[pi]:
                return None
            return "\n".join(
                f"        if (lx::test({self._src_expr(groups[gi])}, bs) && {matches[gi]}(s, bs, bd)) "
                f"return {gi};" for gi in idx)
        claim = phase_switch(claim_body)

        def chain(vals):
            out = str(vals[-1])
            for i in range(len(vals) - 2, -1, -1):
                out = f"(g == {i} ? {vals[i]} : {out})"
            return out
        prio_fn = chain(prios)
        kind_fn = chain([g.kind for g in groups])
        safe_fn = chain(["true" if x else "false" for x in safe])
        # apply: piece move, hop capture, last-action bookkeeping
        hop_cases = []
        for gi, g in enumerate(groups):
            if g.kind == KIND_HOP and (g.capture or self.transient):
                S1, S2 = self._shift_of(g.d1), self._shift_of(g.d2)
                off = str(S1) if S1 == S2 else f"(mover ? {S2} : {S1})"
                hop_cases.append(f"            case {gi}: mid = bs + {off}; cap = {int(g.capture)}; break;")
        hop_sw = ""
        if hop_cases:
            marks = ""
            if self.transient:                 # mechanics.py:347-358
                marks = (f"            {{ const BBW hm = {self._tplane(0)} | om; {self._tplane_set(0, 'hm')} }}\n"
                         f"            if (cap) {{ const BBW cm = {self._tplane(1)} | om; "
                         f"{self._tplane_set(1, 'cm')} }}\n")
            hop_sw = ("        int mid = -1, cap = 0;\n        switch (g) {\n" + "\n".join(hop_cases)
                      + "\n            default: break;\n        }\n"
                      "        if (mid >= 0) {\n            const BBW om = lx::onehot<W>(mid);\n"
                      + marks
                      + "            if (cap) {\n"
                      + self._clear_cells_code("om", "                ") + "\n            }\n        }")
        planes_mv = []
        for t in range(1, self.NPL + 1):
            planes_mv.append(f"        {{ const BBW pl = {self._plane(t)}; const bool bt = lx::test(pl, bs);\n"
                             f"          const BBW q = lx::andnot(pl, os) | lx::sel(bt, lx::bb_zero<W>(), od); "
                             f"{self._plane_set(t, 'q')} }}")
        planes_mv = "\n".join(planes_mv)
        pick_g = ("hint >= 0 ? hint : claim(s, mover, bs, bd)" if all(safe) else
                  "(hint >= 0 && group_safe(hint)) ? hint : claim(s, mover, bs, bd)")
        place_apply = phase_switch(
            lambda pi, idx: (f"                place_write_p{pi}(s, a, mover);\n"
                             f"                return;") if is_place[pi] else None)
        place_legal = phase_switch(
            lambda pi, idx: (f"                return a < {C} && "
                             f"lx::test({groups[idx[0]].legal}, cell_bit(a));") if is_place[pi] else None)

        def enum_body(pi, idx):
            g = groups[idx[0]]
            if is_place[pi]:
                return (f"        {{ const BBW c = {g.legal};\n"
                        f"#pragma unroll\n"
                        f"        for (int w_ = 0; w_ < W; w_++) {{\n"
                        f"            u32 b_ = c.w[w_];\n"
                        f"            while (b_) {{ const int x = 32 * w_ + __ffs(b_) - 1; b_ &= b_ - 1u; "
                        f"f(bit_cell(x)); }}\n"
                        f"        }} }}")
            lines = []
            for gi in idx:
                lines += self._enum_code(gi, groups[gi])
            return "\n".join(lines)
        enum = phase_switch(enum_body)

        # can_move_again: the piece on last_dest, raw group geometry, no
        # priority / must_move (reference mechanics.py:368-403, compiler.py:599-607)
        def cma_body(pi, idx):
            if is_place[pi]:
                return None
            lines = []
            for kind in (KIND_STEP, KIND_HOP, KIND_SLIDE):
                parts = []
                for gi in idx:
                    g = groups[gi]
                    if g.kind != kind:
                        continue
                    S = f"({self._src_expr(g, must=False)} & A_)"
                    if kind == KIND_HOP:
                        f1 = self._count_plane(g, g.d1, S)
                        f2 = self._count_plane(g, g.d2, S)
                    else:   # step and slide: first step along the direction
                        f1 = f"({S} & {self.nb(g.d1, 'E')})"
                        f2 = f"({S} & {self.nb(g.d2, 'E')})"
                    parts.append(f1 if g.symmetric else f"lx::sel(mover != 0, {f1}, {f2})")
                if parts:
                    lines.append(f"        if (kind == {kind}) return lx::any({' | '.join(parts)});")
            return "\n".join(lines) if lines else None
        cma = phase_switch(cma_body)
        code = f"""    static constexpr int MECH = 1, NG = {NG};
    static __device__ __forceinline__ int group_prio(int g) {{ return {prio_fn}; }}
    static __device__ __forceinline__ int group_kind(int g) {{ return {kind_fn}; }}
    static __device__ __forceinline__ bool group_safe(int g) {{ return {safe_fn}; }}
    static __device__ __forceinline__ void count_raw(const St& s, int (&tot)[{NG}]) {{
{pre}
{raw}
    }}
    static __device__ __forceinline__ int count_moves(const St& s, int (&tot)[{NG}]) {{
        count_raw(s, tot);
{filt}
        return n_;
    }}
    static __device__ __forceinline__ int select_move(const St& s, int r, const int (&tot)[{NG}],
                                                      int& hint) {{
{pre}
{sel}
        return -1;
    }}
    static __device__ __forceinline__ int claim(const St& s, int mover_, int bs, int bd) {{
{pre.replace("s.cur", "mover_")}
{claim}
        return -1;
    }}
    static __device__ __forceinline__ bool move_legal(const St& s, int a) {{
{pre}
{place_legal}
        if (a >= {C * C}) return false;
        const int bs = cell_bit(a / {C}), bd = cell_bit(a % {C});
        const int g = claim(s, s.cur, bs, bd);
        if (g < 0) return false;
        {"int tot[NG]; count_raw(s, tot); int minp = " + str(BIG_PRIO) + "; for (int i = 0; i < NG; i++) if (tot[i] > 0 && group_prio(i) < minp) minp = group_prio(i); return group_prio(g) <= minp;" if multi else "return true;"}
    }}
    static __device__ __forceinline__ void apply_move(St& s, int a, int mover, int hint) {{
{place_apply}
        const int src = a / {C}, dst = a % {C};
        const int bs = cell_bit(src), bd = cell_bit(dst);
        const int g = {pick_g};
        if (g < 0) return;                        // unclaimed (unverified) action: no move
        const BBW os = lx::onehot<W>(bs), od = lx::onehot<W>(bd);
        const bool m1 = mover != 0;
        const BBW mine = lx::andnot(m1 ? s.own1 : s.own0, os) | od;
        s.own0 = lx::sel(m1, mine, s.own0);
        s.own1 = lx::sel(m1, s.own1, mine);
{planes_mv}
{hop_sw}
        s.last_kind = group_kind(g); s.last_source = src; s.last_dest = dst; s.last_mover = mover;
        s.ldbp0 = m1 ? s.ldbp0 : dst;
        s.ldbp1 = m1 ? dst : s.ldbp1;
    }}
    template <class F>
    static __device__ __forceinline__ void enum_moves(const St& s, F f) {{
        int tot[NG];
        count_moves(s, tot);
{pre}
{enum}
    }}
    static __device__ __forceinline__ bool can_move_again(const St& s, int mover, int kind) {{
        if (!(s.last_dest >= 0 && s.last_mover == mover)) return false;
        const BBW me = mover ? s.own1 : s.own0;
        const BBW op = mover ? s.own0 : s.own1;
        const BBW E = lx::andnot({self.em.const(self.valid)}, s.own0 | s.own1);
        const BBW A_ = lx::onehot<W>(cell_bit(s.last_dest));
        (void)me; (void)op; (void)E; (void)A_;
{cma}
        return false;
    }}"""
        return code

    def gridworld_code(self, grid):
        """struct Game members of a gridworld game (MECH 2; reference
        mechanics.py:518-608)."""
        player, piece, dirs = grid
        self.grid_dirs = dirs
        NG = len(dirs)
        pid = self.piece_ids[piece]
        mine = self.piece_filter(piece, "me")
        oks = []
        for gi, d in enumerate(dirs):
            k1 = self.em.const(self._walk_ok(d, 1))
            oks.append(f"        tot[{gi}] = (lx::test({k1}, x) && lx::test(E, x + {self._shift_of(d)})) ? 1 : 0;")
        oks = "\n".join(oks)
        sums = " + ".join(f"tot[{gi}]" for gi in range(NG))
        sel = "\n".join(f"        if (r < tot[{gi}]) {{ hint = {gi}; return {gi}; }}\n        r -= tot[{gi}];"
                        for gi in range(NG))
        offs = ", ".join(str(self._shift_of(d)) for d in dirs)
        set_t = ""
        if self.piece_mode == "planes" and pid >= 1:
            set_t = f"\n        {{ BBW pl = {self._plane(pid)}; lx::setbit(pl, bd); {self._plane_set(pid, 'pl')} }}"
        planes_clear = ""
        if self.NPL:
            planes_clear = "\n" + "\n".join(
                f"        {{ const BBW pl = lx::andnot({self._plane(t)}, os); {self._plane_set(t, 'pl')} }}"
                for t in range(1, self.NPL + 1))
        pre = "\n".join(self._mv_prelude())
        return f"""    static constexpr int MECH = 2, NG = {NG};
    static __device__ __forceinline__ int walker(const St& s, int mover) {{
        const BBW me = mover ? s.own1 : s.own0;
        const BBW m = {mine};
        return lx::any(m) ? lx::select_bit(m, 0) : cell_bit(0);     // argmax of an all-false row is 0
    }}
    static __device__ __forceinline__ void count_raw(const St& s, int (&tot)[{NG}]) {{
{pre}
        const int x = walker(s, mover);
{oks}
        if (s.phase >= NPHASE) {{                 // dead phase after once_through: no moves
#pragma unroll
            for (int i = 0; i < {NG}; i++) tot[i] = 0;
        }}
    }}
    static __device__ __forceinline__ int count_moves(const St& s, int (&tot)[{NG}]) {{
        count_raw(s, tot);
        return {sums};
    }}
    static __device__ __forceinline__ int select_move(const St& s, int r, const int (&tot)[{NG}],
                                                      int& hint) {{
{sel}
        hint = -1;
        return -1;
    }}
    static __device__ __forceinline__ bool move_legal(const St& s, int a) {{
        int tot[NG];
        count_raw(s, tot);
        for (int i = 0; i < NG; i++) if (i == a) return tot[i] > 0;
        return false;
    }}
    static __device__ __forceinline__ void apply_move(St& s, int a, int mover, int hint) {{
        (void)hint;
        int tot[NG];
        count_raw(s, tot);                        // s.cur is the mover during the ply
        bool ok = false;
        for (int i = 0; i < NG; i++) if (i == a) ok = tot[i] > 0;
        if (!ok) return;                          // illegal (unverified) direction: no move
        const int off[{NG}] = {{{offs}}};
        int o = 0;
        for (int i = 0; i < NG; i++) if (i == a) o = off[i];
        const int bs = walker(s, mover), bd = bs + o;
        const BBW os = lx::onehot<W>(bs), od = lx::onehot<W>(bd);
        const bool m1 = mover != 0;
        s.own0 = lx::andnot(s.own0, os); s.own1 = lx::andnot(s.own1, os);{planes_clear}
        s.own0 = lx::sel(m1, s.own0 | od, s.own0);
        s.own1 = lx::sel(m1, s.own1, s.own1 | od);{set_t}
        const int src = bit_cell(bs), dst = bit_cell(bd);
        s.last_kind = {KIND_STEP}; s.last_source = src; s.last_dest = dst; s.last_mover = mover;
        s.ldbp0 = m1 ? s.ldbp0 : dst;
        s.ldbp1 = m1 ? dst : s.ldbp1;
    }}
    template <class F>
    static __device__ __forceinline__ void enum_moves(const St& s, F f) {{
        int tot[NG];
        count_raw(s, tot);
        for (int i = 0; i < NG; i++) if (tot[i]) f(i);
    }}
    static __device__ __forceinline__ bool can_move_again(const St& s, int mover, int kind) {{
        if (kind != {KIND_STEP}) return false;
        int tot[NG];
        St t_ = s;
        t_.cur = mover;
        return count_moves(t_, tot) > 0;
    }}"""

    def placement_stubs(self):
        """Movement entry points of a placement game (never called; the
        kernels dispatch on MECH with if constexpr in non-template code)."""
        return """    static constexpr int NG = 1;
    static __device__ __forceinline__ int count_moves(const St&, int (&tot)[1]) { tot[0] = 0; return 0; }
    static __device__ __forceinline__ int select_move(const St&, int, const int (&)[1], int& hint) { hint = -1; return -1; }
    static __device__ __forceinline__ bool move_legal(const St&, int) { return false; }
    static __device__ __forceinline__ void apply_move(St&, int, int, int) {}
    template <class F>
    static __device__ __forceinline__ void enum_moves(const St&, F) {}
    static __device__ __forceinline__ bool can_move_again(const St&, int, int) { return false; }"""

    def movement_stubs(self):
        """Placement entry points of a movement game (never called)."""
        return """    static __device__ __forceinline__ BBW legal(const St&) { return lx::bb_zero<W>(); }
    static __device__ __forceinline__ void write_place(St&, int, int, int) {}"""
