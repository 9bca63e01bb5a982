/*
 * ludax_oracle.c -- CPU ORACLE FOR PARITY TESTS.  TEST INFRASTRUCTURE ONLY.
 *
 * A scalar, cell-array restatement of the reference's rollout hot path
 * (reference: /root/reference/pkg/src/boardlang/, the numpy "boardlang"
 * re-implementation of Ludax) for the eleven corpus games: placement games
 * (mechanics.py:415-515) and, in the movement section below, the movement /
 * gridworld games (mechanics.py:44-404, 518-608) with their per-source count
 * formulation of legality and sampling.  It works on the
 * reference's own structure-of-arrays GameState layout (state.py:78-130:
 * int8 boards with -1 = empty, int32 move_count, ...), so its outputs can be
 * hashed with the reference's digest and compared field by field.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library, and only as the checker / the timed CPU reference arm.
 * The product path (paper_2506_22609_b200/) never links or calls it.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/, generator oracle/gen_golden.py).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXC 384
#define MAXW 1100

enum { FAM_GRID = 0, FAM_HEXRECT = 1, FAM_HEXAGON = 2 };
enum { DEST_EMPTY = 0, DEST_C4 = 1, DEST_CENTER = 2 };
enum { EFF_NONE = 0, EFF_REVERSI = 1, EFF_PENTE = 2 };
enum { END_LINE = 0, END_FULL = 1, END_CONN = 2, END_PASSED_BOTH = 3, END_SCORE_GE = 4, END_LINE_LOSE = 5,
       END_NO_LEGAL = 6, END_LAST_MOVE_IN = 7, END_LINE_EXCL = 8 };
enum { MECH_PLACE = 0, MECH_MOVE = 1, MECH_GRID = 2 };
enum { K_PLACE = 0, K_STEP = 1, K_HOP = 2, K_SLIDE = 3, K_PASS = 4 };    /* state.py:23-31 */
enum { OVER_ANY = 0, OVER_OPP = 1, OVER_MOVER = 2 };
#define MAXG 16
enum { RES_MOVER_WIN = 0, RES_DRAW = 1, RES_BY_SCORE = 2, RES_MOVER_LOSE = 3 };
enum { ST_OK = 0, ST_ILLEGAL = 1, ST_TERMINAL = 2, ST_EMPTY_MASK = 3 };

/* --- rng.py:12-42 --------------------------------------------------------- */
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t hash2(uint64_t a, uint64_t b) {        /* hash_key(a, b) */
    return mix64(mix64(0x243F6A8885A308D3ull ^ a) ^ b);
}
static inline double uniform2(uint64_t seed, uint64_t mc) {   /* uniform(seed, mc) */
    return (double)(hash2(seed, mc) >> 11) * (1.0 / 9007199254740992.0);
}

typedef struct {
    int game, C, A, has_pass, pass_index, rows, cols, family;
    int ndirs;
    int16_t nbr[8][MAXC + 1];      /* topology.py:182-190, board direction order */
    int dir_dx[8], dir_dy[8];
    int bottom_row_first;
    int center;
    uint8_t edge[4][MAXC];         /* top, bottom, left, right (topology.py:224-233) */
    /* StateLayout (compiler.py:98-152) */
    int L_scores, L_passing, L_last, L_conn, L_phase;
    /* phases (compiler.py:233-267) */
    int nphase;
    int once[3], olen[3], order[3][2], force_pass[3], dest[3], result_cust[3], effect[3];
    /* end rules in order (compiler.py:283-286) */
    int nend;
    int end_kind[4], end_arg[4], end_gate[4], end_ea[4], end_eb[4], end_res[4], end_anch[4];
    /* line windows for "any" orientation (topology.py:319-359) */
    struct {
        int len, nwin, exact;
        int16_t win[MAXW][5];
        int16_t before[MAXW], after[MAXW];       /* extension cells (topology.py:348-352) */
    } lt[2];                                      /* one table per line end rule */
    int nlt;
    /* custodial walk directions: each axis then its inverse (exprs.py:244-251) */
    int ncust;
    int cust_dir[8];
    int ray_max;                   /* stacked ray length L (exprs.py:386-396) */
    /* movement games (compiler.py:311-327; mechanics.py:44-82) */
    int mech, L_must, needs_next, multi_prio;
    int ng;
    struct { int kind, piece, prio, d[2], over, capture, L; } grp[MAXG];
    int nstart, start_cell[64], start_player[64], start_piece[64];
    int promote, promote_from, promote_to;                 /* (promote a b (edge forward)) */
    int extra_hop;                 /* (if (and (action_was mover hop) (can_move_again hop)) (extra_turn mover same_piece:true)) */
    int cap_custodial, corner_cust;                        /* Dai Hasami Shogi effects */
    int ncorner, corner[4][3];
    uint8_t end_mask[4][MAXC];     /* last_move_in masks / line exclusions per end rule */
    int grid_piece, grid_ndir, grid_dir[8];
} orc_game;

typedef struct {
    int8_t *board_piece, *board_owner, *current_player;
    int32_t *move_count;
    uint8_t *terminated, *truncated;
    int8_t *outcome;
    uint64_t *seeds;
    int32_t *scores;
    int16_t *pass_streak;
    uint8_t *pass_flags;
    int8_t *last_mover, *last_kind;
    int16_t *last_source, *last_dest, *last_dest_by_player, *comp_labels;
    int8_t *phase;
    int16_t *must_move;
} orc_soa;

static const char *GRID_DIRS[8] = {"up", "down", "left", "right", "up_left", "up_right",
                                   "down_left", "down_right"};
static const int GRID_D[8][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {-1, -1}, {-1, 1},
                                 {1, -1}, {1, 1}};
static const int HEXR_D[6][2] = {{0, -1}, {0, 1}, {-1, 0}, {1, 0}, {-1, 1}, {1, -1}};
/* hex_rectangle order: left, right, up, down, up_right, down_left */

static int dir_index_grid(const char *n) {
    for (int i = 0; i < 8; i++) if (!strcmp(GRID_DIRS[i], n)) return i;
    return -1;
}

static void build_topology(orc_game *g, int family, int rows, int cols) {
    g->family = family; g->rows = rows; g->cols = cols; g->C = rows * cols;
    g->ndirs = family == FAM_GRID ? 8 : 6;
    int C = g->C;
    for (int d = 0; d < g->ndirs; d++) {
        int dr = family == FAM_GRID ? GRID_D[d][0] : HEXR_D[d][0];
        int dc = family == FAM_GRID ? GRID_D[d][1] : HEXR_D[d][1];
        g->dir_dx[d] = dr; g->dir_dy[d] = dc;
        for (int i = 0; i <= C; i++) g->nbr[d][i] = (int16_t)C;
        for (int r = 0; r < rows; r++)
            for (int c = 0; c < cols; c++) {
                int rr = r + dr, cc = c + dc;
                if (rr >= 0 && rr < rows && cc >= 0 && cc < cols)
                    g->nbr[d][r * cols + c] = (int16_t)(rr * cols + cc);
            }
    }
    for (int i = 0; i < C; i++) {
        int r = i / cols, c = i % cols;
        g->edge[0][i] = r == 0; g->edge[1][i] = r == rows - 1;
        g->edge[2][i] = c == 0; g->edge[3][i] = c == cols - 1;
    }
    /* topology.py:247-257 centre: middle row(s) x middle column(s); the
       config boards with a centre mask (19x19) have odd sides */
    g->center = (rows / 2) * cols + cols / 2;
}

static int ray_len(const orc_game *g, int d) {
    int best = 0;
    for (int s = 0; s < g->C; s++) {
        int k = 0, x = s;
        while (g->nbr[d][x] != g->C) { x = g->nbr[d][x]; k++; }
        if (k > best) best = k;
    }
    return best;
}

/* hexagon boards (topology.py:134-150): axial (q, r), rows r = -R..R, cells
   row-major; directions left, right, up_left, up_right, down_left, down_right */
static const int HEXA_D[6][2] = {{-1, 0}, {1, 0}, {0, -1}, {1, -1}, {-1, 1}, {0, 1}};

static void build_hexagon(orc_game *g, int diameter) {
    int R = (diameter - 1) / 2, n = 0;
    static int qs[MAXC], rs[MAXC];
    g->family = FAM_HEXAGON; g->rows = g->cols = diameter; g->ndirs = 6;
    for (int r = -R; r <= R; r++) {
        int lo = -R > -R - r ? -R : -R - r, hi = R < R - r ? R : R - r;
        for (int q = lo; q <= hi; q++) { qs[n] = q; rs[n] = r; n++; }
    }
    g->C = n;
    for (int d = 0; d < 6; d++) {
        for (int i = 0; i <= n; i++) g->nbr[d][i] = (int16_t)n;
        for (int i = 0; i < n; i++)
            for (int j = 0; j < n; j++)
                if (qs[j] == qs[i] + HEXA_D[d][0] && rs[j] == rs[i] + HEXA_D[d][1]) g->nbr[d][i] = (int16_t)j;
    }
}

/* windows of `len` cells along each axis of orientation "any", per start
   cell (topology.py:319-359): grids right, down, down_right, down_left;
   hexagons right, down_left, down_right.  Returns the table index. */
static int build_lines(orc_game *g, int len, int exact) {
    static const char *axes[4] = {"right", "down", "down_right", "down_left"};
    static const char *inv_axes[4] = {"left", "up", "up_left", "up_right"};
    static const int hex_axes[3] = {1, 4, 5}, hex_inv[3] = {0, 3, 2};
    int t = g->nlt++;
    g->lt[t].len = len; g->lt[t].nwin = 0; g->lt[t].exact = exact;
    int naxes = g->family == FAM_HEXAGON ? 3 : 4;
    for (int a = 0; a < naxes; a++) {
        int d = g->family == FAM_HEXAGON ? hex_axes[a] : dir_index_grid(axes[a]);
        int di = g->family == FAM_HEXAGON ? hex_inv[a] : dir_index_grid(inv_axes[a]);
        for (int s = 0; s < g->C; s++) {
            int cells[8], k = 1; cells[0] = s;
            while (k < len && g->nbr[d][cells[k - 1]] != g->C) { cells[k] = g->nbr[d][cells[k - 1]]; k++; }
            if (k == len) {
                int w = g->lt[t].nwin++;
                for (int j = 0; j < len; j++) g->lt[t].win[w][j] = (int16_t)cells[j];
                g->lt[t].before[w] = g->nbr[di][s];
                g->lt[t].after[w] = g->nbr[d][cells[len - 1]];
            }
        }
    }
    return t;
}

/* windows along explicit grid axes (orientation "orthogonal": right, down) */
static int build_lines_axes(orc_game *g, int len, int naxes, const char **axes, const char **inv) {
    int t = g->nlt++;
    g->lt[t].len = len; g->lt[t].nwin = 0; g->lt[t].exact = 0;
    for (int a = 0; a < naxes; a++) {
        int d = dir_index_grid(axes[a]), di = dir_index_grid(inv[a]);
        for (int s = 0; s < g->C; s++) {
            int cells[8], k = 1; cells[0] = s;
            while (k < len && g->nbr[d][cells[k - 1]] != g->C) { cells[k] = g->nbr[d][cells[k - 1]]; k++; }
            if (k == len) {
                int w = g->lt[t].nwin++;
                for (int j = 0; j < len; j++) g->lt[t].win[w][j] = (int16_t)cells[j];
                g->lt[t].before[w] = g->nbr[di][s];
                g->lt[t].after[w] = g->nbr[d][cells[len - 1]];
            }
        }
    }
    return t;
}

static void build_custodial_n(orc_game *g, int naxes) {
    static const char *axes[4] = {"right", "down", "down_right", "down_left"};
    static const char *inv[4] = {"left", "up", "up_left", "up_right"};
    g->ncust = 0;
    for (int a = 0; a < naxes; a++) {
        g->cust_dir[g->ncust++] = dir_index_grid(axes[a]);
        g->cust_dir[g->ncust++] = dir_index_grid(inv[a]);
    }
    g->ray_max = 0;
    for (int i = 0; i < g->ncust; i++) {
        int l = ray_len(g, g->cust_dir[i]);
        if (l > g->ray_max) g->ray_max = l;
    }
}

static void build_custodial(orc_game *g) { build_custodial_n(g, 4); }

static void add_group(orc_game *g, int kind, int piece, int prio, const char *d1, const char *d2,
                      int over, int capture) {
    int k = g->ng++;
    g->grp[k].kind = kind; g->grp[k].piece = piece; g->grp[k].prio = prio;
    g->grp[k].d[0] = dir_index_grid(d1); g->grp[k].d[1] = dir_index_grid(d2);
    g->grp[k].over = over; g->grp[k].capture = capture;
    int l0 = ray_len(g, g->grp[k].d[0]), l1 = ray_len(g, g->grp[k].d[1]);
    if (l0 < 1) l0 = 1;
    if (l1 < 1) l1 = 1;
    g->grp[k].L = l0 > l1 ? l0 : l1;                  /* mechanics.py:67-80 (distance 0) */
    if (k > 0 && g->grp[k].prio != g->grp[0].prio) g->multi_prio = 1;
}

static void add_start(orc_game *g, int player, int piece, const int *cells, int n) {
    for (int j = 0; j < n; j++) {
        g->start_cell[g->nstart] = cells[j]; g->start_player[g->nstart] = player;
        g->start_piece[g->nstart] = piece; g->nstart++;
    }
}

static const char *DIAG[4] = {"up_left", "up_right", "down_left", "down_right"};
static const char *ORTH[4] = {"up", "down", "left", "right"};

/* movement corpus games: groups in the reference's order (compiler.py:311-327;
   direction_pairs, mechanics.py:25-41) */
static int new_movement_game(orc_game *g, const char *name) {
    if (!strcmp(name, "english_draughts")) {          /* games/english_draughts.ldx */
        static const int p1[12] = {40, 42, 44, 46, 49, 51, 53, 55, 56, 58, 60, 62};
        static const int p2[12] = {1, 3, 5, 7, 8, 10, 12, 14, 17, 19, 21, 23};
        g->game = 10; build_topology(g, FAM_GRID, 8, 8); g->mech = MECH_MOVE;
        add_start(g, 0, 0, p1, 12); add_start(g, 1, 0, p2, 12);
        /* pawn forward_left / forward_right: P1 up -> up_left/up_right, P2 down -> down_right/down_left */
        add_group(g, K_HOP, 0, 0, "up_left", "down_right", OVER_OPP, 1);
        add_group(g, K_HOP, 0, 0, "up_right", "down_left", OVER_OPP, 1);
        add_group(g, K_STEP, 0, 1, "up_left", "down_right", OVER_ANY, 0);
        add_group(g, K_STEP, 0, 1, "up_right", "down_left", OVER_ANY, 0);
        for (int k = 0; k < 4; k++) add_group(g, K_HOP, 1, 0, DIAG[k], DIAG[k], OVER_OPP, 1);
        for (int k = 0; k < 4; k++) add_group(g, K_STEP, 1, 1, DIAG[k], DIAG[k], OVER_ANY, 0);
        g->promote = 1; g->promote_from = 0; g->promote_to = 1;
        g->extra_hop = 1;
        g->L_must = 1; g->L_last = 1; g->needs_next = 1;
        g->nend = 1;
        g->end_kind[0] = END_NO_LEGAL; g->end_res[0] = RES_MOVER_WIN;
    } else if (!strcmp(name, "dai_hasami_shogi")) {   /* games/dai_hasami_shogi.ldx */
        int p1[18], p2[18];
        for (int k = 0; k < 18; k++) { p1[k] = 63 + k; p2[k] = k; }
        g->game = 11; build_topology(g, FAM_GRID, 9, 9); g->mech = MECH_MOVE;
        add_start(g, 0, 0, p1, 18); add_start(g, 1, 0, p2, 18);
        for (int k = 0; k < 4; k++) add_group(g, K_SLIDE, 0, 0, ORTH[k], ORTH[k], OVER_ANY, 0);
        for (int k = 0; k < 4; k++) add_group(g, K_HOP, 0, 0, ORTH[k], ORTH[k], OVER_ANY, 0);
        build_custodial_n(g, 2);                     /* orientation orthogonal: right, down */
        g->cap_custodial = 1; g->corner_cust = 1;
        /* corners top_left, top_right, bottom_left, bottom_right with their
           (up, down, left, right) neighbours (exprs.py:381-392) */
        static const int cs[4] = {0, 8, 72, 80};
        for (int k = 0; k < 4; k++) {
            int c = cs[k], m = 0;
            g->corner[k][0] = c;
            for (int d = 0; d < 4; d++) if (g->nbr[d][c] != g->C) g->corner[k][1 + m++] = g->nbr[d][c];
        }
        g->ncorner = 4;
        g->L_last = 1;
        static const char *ax[2] = {"right", "down"}, *iv[2] = {"left", "up"};
        build_lines_axes(g, 5, 2, ax, iv);
        g->nend = 2;
        g->end_kind[0] = END_LINE_EXCL; g->end_arg[0] = 0; g->end_gate[0] = 0; g->end_res[0] = RES_MOVER_WIN;
        g->end_kind[1] = END_LINE_EXCL; g->end_arg[1] = 0; g->end_gate[1] = 1; g->end_res[1] = RES_MOVER_WIN;
        for (int c = 0; c < g->C; c++) {
            int r = c / 9;
            g->end_mask[0][c] = r == 7 || r == 8;     /* exclude:((row 7) (row 8)) */
            g->end_mask[1][c] = r == 0 || r == 1;
        }
    } else if (!strcmp(name, "wolf_and_sheep")) {     /* games/wolf_and_sheep.ldx */
        static const int sheep[4] = {56, 58, 60, 62}, wolf[1] = {3};
        g->game = 12; build_topology(g, FAM_GRID, 8, 8); g->mech = MECH_MOVE;
        add_start(g, 0, 0, sheep, 4); add_start(g, 1, 1, wolf, 1);
        add_group(g, K_STEP, 0, 0, "up_left", "down_right", OVER_ANY, 0);
        add_group(g, K_STEP, 0, 0, "up_right", "down_left", OVER_ANY, 0);
        for (int k = 0; k < 4; k++) add_group(g, K_STEP, 1, 0, DIAG[k], DIAG[k], OVER_ANY, 0);
        g->L_last = 1; g->needs_next = 1;
        g->nend = 2;
        g->end_kind[0] = END_LAST_MOVE_IN; g->end_gate[0] = 1; g->end_res[0] = RES_MOVER_WIN;
        for (int c = 0; c < g->C; c++) g->end_mask[0][c] = g->edge[1][c];     /* edge bottom */
        g->end_kind[1] = END_NO_LEGAL; g->end_res[1] = RES_MOVER_WIN;
    } else if (!strcmp(name, "gridworld")) {          /* games/gridworld.ldx */
        static const int walker[1] = {0};
        g->game = 13; build_topology(g, FAM_GRID, 4, 4); g->mech = MECH_GRID;
        add_start(g, 0, 0, walker, 1);
        g->olen[0] = 1; g->order[0][0] = 0;            /* (repeat (P1)) */
        g->grid_piece = 0; g->grid_ndir = 4;
        for (int k = 0; k < 4; k++) g->grid_dir[k] = k; /* up, down, left, right */
        g->L_last = 1;
        g->nend = 2;
        g->end_kind[0] = END_LAST_MOVE_IN; g->end_gate[0] = -1; g->end_res[0] = RES_MOVER_WIN;
        g->end_mask[0][15] = 1;                         /* region target */
        g->end_kind[1] = END_LAST_MOVE_IN; g->end_gate[1] = -1; g->end_res[1] = RES_MOVER_LOSE;
        g->end_mask[1][5] = g->end_mask[1][7] = g->end_mask[1][11] = g->end_mask[1][12] = 1;
    } else {
        return 0;
    }
    if (g->mech == MECH_MOVE) g->A = g->C * g->C;
    else g->A = g->grid_ndir;
    g->pass_index = -1;
    return 1;
}

orc_game *orc_game_new(const char *name) {
    orc_game *g = (orc_game *)calloc(1, sizeof(orc_game));
    g->nphase = 1; g->olen[0] = 2; g->order[0][0] = 0; g->order[0][1] = 1;
    if (!strcmp(name, "tic_tac_toe")) {                 /* games/tic_tac_toe.ldx */
        g->game = 0; build_topology(g, FAM_GRID, 3, 3); build_lines(g, 3, 0);
        g->nend = 2;
        g->end_kind[0] = END_LINE; g->end_arg[0] = 0; g->end_anch[0] = 0; g->end_res[0] = RES_MOVER_WIN;
        g->end_kind[1] = END_FULL; g->end_res[1] = RES_DRAW;
    } else if (!strcmp(name, "connect_four")) {         /* games/connect_four.ldx */
        g->game = 1; build_topology(g, FAM_GRID, 6, 7); build_lines(g, 4, 0);
        g->dest[0] = DEST_C4; g->L_last = 1;
        g->nend = 2;
        /* 69 windows * 4 > 128: anchored at last_dest (compiler.py:28,122-135) */
        g->end_kind[0] = END_LINE; g->end_arg[0] = 0; g->end_anch[0] = 1; g->end_res[0] = RES_MOVER_WIN;
        g->end_kind[1] = END_FULL; g->end_res[1] = RES_DRAW;
    } else if (!strcmp(name, "hex")) {                  /* games/hex.ldx */
        g->game = 2; build_topology(g, FAM_HEXRECT, 11, 11);
        g->L_conn = 1;
        g->nend = 2;
        g->end_kind[0] = END_CONN; g->end_gate[0] = 0; g->end_ea[0] = 0; g->end_eb[0] = 1; g->end_res[0] = RES_MOVER_WIN;
        g->end_kind[1] = END_CONN; g->end_gate[1] = 1; g->end_ea[1] = 2; g->end_eb[1] = 3; g->end_res[1] = RES_MOVER_WIN;
    } else if (!strcmp(name, "reversi")) {              /* games/reversi.ldx */
        g->game = 3; build_topology(g, FAM_GRID, 8, 8); build_custodial(g);
        g->has_pass = 1; g->force_pass[0] = 1; g->result_cust[0] = 1; g->effect[0] = EFF_REVERSI;
        g->L_scores = 1; g->L_passing = 1; g->L_last = 1;
        g->nend = 1;
        g->end_kind[0] = END_PASSED_BOTH; g->end_res[0] = RES_BY_SCORE;
    } else if (!strcmp(name, "pente")) {                /* games/pente.ldx */
        g->game = 4; build_topology(g, FAM_GRID, 19, 19); build_lines(g, 5, 0); build_custodial(g);
        g->nphase = 2;
        g->once[0] = 1; g->olen[0] = 1; g->order[0][0] = 0; g->dest[0] = DEST_CENTER;
        g->once[1] = 0; g->olen[1] = 2; g->order[1][0] = 1; g->order[1][1] = 0; g->dest[1] = DEST_EMPTY;
        g->effect[1] = EFF_PENTE;
        g->L_scores = 1; g->L_last = 1; g->L_phase = 1;
        g->nend = 3;
        g->end_kind[0] = END_LINE; g->end_arg[0] = 0; g->end_anch[0] = 1; g->end_res[0] = RES_MOVER_WIN;
        g->end_kind[1] = END_SCORE_GE; g->end_arg[1] = 10; g->end_res[1] = RES_MOVER_WIN;
        g->end_kind[2] = END_FULL; g->end_res[2] = RES_DRAW;
    } else if (!strcmp(name, "gomoku")) {              /* corpus: games/gomoku.ldx */
        g->game = 5; build_topology(g, FAM_GRID, 15, 15); build_lines(g, 5, 1);
        g->L_last = 1;
        g->nend = 2;
        g->end_kind[0] = END_LINE; g->end_arg[0] = 0; g->end_anch[0] = 1; g->end_res[0] = RES_MOVER_WIN;
        g->end_kind[1] = END_FULL; g->end_res[1] = RES_DRAW;
    } else if (!strcmp(name, "yavalath")) {            /* corpus: games/yavalath.ldx */
        g->game = 6; build_hexagon(g, 9); build_lines(g, 4, 0); build_lines(g, 3, 0);
        g->L_last = 1;
        g->nend = 3;
        g->end_kind[0] = END_LINE; g->end_arg[0] = 0; g->end_anch[0] = 1; g->end_res[0] = RES_MOVER_WIN;
        g->end_kind[1] = END_LINE_LOSE; g->end_arg[1] = 1; g->end_anch[1] = 1; g->end_res[1] = RES_MOVER_LOSE;
        g->end_kind[2] = END_FULL; g->end_res[2] = RES_DRAW;
    } else {
        if (new_movement_game(g, name)) return g;
        free(g);
        return NULL;
    }
    g->A = g->C + (g->has_pass ? 1 : 0);
    g->pass_index = g->has_pass ? g->C : -1;
    return g;
}

void orc_game_free(orc_game *g) { free(g); }
int orc_num_cells(const orc_game *g) { return g->C; }
int orc_num_actions(const orc_game *g) { return g->A; }
/* layout bits: 1 scores, 2 passing, 4 last_action, 8 connectivity, 16 phase, 32 must_move */
int orc_layout(const orc_game *g) {
    return g->L_scores | (g->L_passing << 1) | (g->L_last << 2) | (g->L_conn << 3) | (g->L_phase << 4)
        | (g->L_must << 5);
}
int orc_mechanics(const orc_game *g) { return g->mech; }

/* --- per-env views --------------------------------------------------------- */
typedef struct { const orc_game *g; orc_soa *s; int64_t i; int8_t *own; int8_t *pc; } env_t;

static inline env_t env_of(const orc_game *g, orc_soa *s, int64_t i) {
    env_t e = {g, s, i, s->board_owner + i * g->C, s->board_piece + i * g->C};
    return e;
}
static inline int phase_of(const env_t *e) { return e->s->phase ? e->s->phase[e->i] : 0; }

/* Reversi placement result: exprs.py:334-378 (would_custodial), i.e. a run of
   >= 1 opponent discs from the candidate followed by a mover disc. */
static int would_flank(const env_t *e, int c, int side) {
    const orc_game *g = e->g;
    int tgt = 1 - side;
    for (int k = 0; k < g->ncust; k++) {
        int d = g->cust_dir[k];
        int x = g->nbr[d][c], run = 0;
        while (x != g->C && e->own[x] == tgt && e->pc[x] == 0) { run++; x = g->nbr[d][x]; }
        if (run >= 1 && run <= g->ray_max - 1 && x != g->C && e->own[x] == side) return 1;
    }
    return 0;
}

/* PlacementMechanics.legal_cells (mechanics.py:432-439) */
static int legal_cells(const env_t *e, int mover, uint8_t *out) {
    const orc_game *g = e->g;
    int p = phase_of(e), n = 0;
    int down = g->family == FAM_GRID ? dir_index_grid("down") : 3;
    for (int c = 0; c < g->C; c++) {
        int ok = e->own[c] < 0;
        if (ok && g->dest[p] == DEST_C4) {
            /* (or (edge bottom) (adjacent (occupied) direction:up)):
               exprs.py:178-195 reads the occupancy of the down-neighbour */
            int nb = g->nbr[down][c];
            ok = g->edge[1][c] || (nb != g->C && e->own[nb] >= 0);
        } else if (ok && g->dest[p] == DEST_CENTER) {
            ok = c == g->center;
        }
        if (ok && g->result_cust[p]) ok = would_flank(e, c, mover);
        out[c] = (uint8_t)ok;
        n += ok;
    }
    return n;
}

/* compiler.py:394-428 */
static int legal_count_and_mask(const env_t *e, uint8_t *cells, uint8_t *mask_out) {
    const orc_game *g = e->g;
    int n = legal_cells(e, e->s->current_player[e->i], cells);
    int p = phase_of(e);
    int term = e->s->terminated[e->i];
    if (mask_out) {
        for (int c = 0; c < g->C; c++) mask_out[c] = term ? 0 : cells[c];
        if (g->has_pass) mask_out[g->C] = (!term && g->force_pass[p] && n == 0);
    }
    int total = n;
    if (g->has_pass && g->force_pass[p] && n == 0) total = 1;
    return term ? 0 : total;
}

/* compiler.py:430-446 + mechanics.py:488-492 */
static int64_t sample_one(const env_t *e, double u, uint8_t *cells) {
    const orc_game *g = e->g;
    if (e->s->terminated[e->i]) return -1;
    int n = legal_cells(e, e->s->current_player[e->i], cells);
    int p = phase_of(e);
    int64_t r = (int64_t)(u * (double)n);
    int64_t hi = n - 1 > 0 ? n - 1 : 0;
    if (r > hi) r = hi;
    if (n == 0) return (g->has_pass && g->force_pass[p]) ? g->pass_index : -1;
    int64_t k = 0;
    for (int c = 0; c < g->C; c++)
        if (cells[c]) { if (k == r) return c; k++; }
    return -1;
}

/* connectivity.py:16-45 (labels stay min-index of each component) */
static void place_update(env_t *e, int cell) {
    const orc_game *g = e->g;
    int16_t *lab = e->s->comp_labels + e->i * g->C;
    int owner = e->own[cell];
    int16_t nl[8]; int ok[8];
    int newl = cell;
    for (int d = 0; d < g->ndirs; d++) {
        int nb = g->nbr[d][cell];
        ok[d] = nb != g->C && e->own[nb] == owner;
        nl[d] = nb != g->C ? lab[nb] : -1;
        if (ok[d] && nl[d] >= 0 && nl[d] < newl) newl = nl[d];
    }
    lab[cell] = (int16_t)newl;
    for (int d = 0; d < g->ndirs; d++) {
        if (ok[d] && nl[d] != newl && nl[d] >= 0) {
            int16_t old = nl[d];
            for (int c = 0; c < g->C; c++) if (lab[c] == old) lab[c] = (int16_t)newl;
        }
    }
}

/* exprs.py:629-652 connected(): some component of `side` touches both edges */
static int connected2(const env_t *e, int side, int ea, int eb) {
    const orc_game *g = e->g;
    const int16_t *lab = e->s->comp_labels + e->i * g->C;
    static __thread uint8_t hit[MAXC];
    memset(hit, 0, g->C);
    for (int c = 0; c < g->C; c++)
        if (e->own[c] == side && g->edge[ea][c] && lab[c] >= 0) hit[lab[c]] = 1;
    for (int c = 0; c < g->C; c++)
        if (e->own[c] == side && g->edge[eb][c] && lab[c] >= 0 && hit[lab[c]]) return 1;
    return 0;
}

/* _LineTables.satisfied / compile_line_anchored_exists (exprs.py:433-535) */
static int line_sat(const env_t *e, int side, int anchored, int t) {
    const orc_game *g = e->g;
    int dest = g->C, len = g->lt[t].len;
    if (anchored) {
        int ld = e->s->last_dest[e->i];
        if (ld >= 0 && e->s->last_mover[e->i] == side) dest = ld; else return 0;
    }
    for (int w = 0; w < g->lt[t].nwin; w++) {
        int through = !anchored, ok = 1;
        for (int j = 0; j < len; j++) through |= g->lt[t].win[w][j] == dest;
        if (!through) continue;
        for (int j = 0; j < len && ok; j++) {
            int c = g->lt[t].win[w][j];
            ok = e->own[c] == side && e->pc[c] == 0;
        }
        if (ok && g->lt[t].exact) {       /* exprs.py:444-448: extensions not the side's */
            int b = g->lt[t].before[w], a = g->lt[t].after[w];
            if (b != g->C && e->own[b] == side && e->pc[b] == 0) ok = 0;
            if (a != g->C && e->own[a] == side && e->pc[a] == 0) ok = 0;
        }
        if (ok) return 1;
    }
    return 0;
}

/* anchored custodial walk from the placed cell (exprs.py:254-292):
   marks the run when it is flanked; length = 0 means "any". */
static int custodial_from(const env_t *e, int anchor, int side, int length, int16_t *mark) {
    const orc_game *g = e->g;
    int tgt = 1 - side, L = g->ray_max, m = 0;
    for (int k = 0; k < g->ncust; k++) {
        int d = g->cust_dir[k];
        int x = g->nbr[d][anchor], run = 0;
        int16_t cells[32];
        while (x != g->C && e->own[x] == tgt && e->pc[x] == 0) { cells[run++] = (int16_t)x; x = g->nbr[d][x]; }
        int ok = run >= 1 && run < L && x != g->C && e->own[x] == side;
        if (length > 0) ok = ok && run == length;
        if (ok) for (int j = 0; j < run; j++) mark[m++] = cells[j];
    }
    return m;
}

static int count_owned(const env_t *e, int side) {
    int n = 0;
    for (int c = 0; c < e->g->C; c++) n += e->own[c] == side;
    return n;
}

/* CompiledGame.step_into for one live row (compiler.py:456-580) */
static int step_one(env_t *e, int64_t action, int verify, uint8_t *scratch) {
    const orc_game *g = e->g;
    orc_soa *s = e->s;
    int64_t i = e->i;
    int mover = s->current_player[i];
    int phase = phase_of(e);
    int pos = 0;
    for (int k = 0; k < g->olen[phase]; k++) if (g->order[phase][k] == mover) { pos = k; break; }
    int is_pass = g->has_pass && action == g->pass_index;
    if (is_pass) {
        if (verify) {
            int n = legal_cells(e, mover, scratch);
            if (n > 0 || !g->force_pass[phase]) return ST_ILLEGAL;
        }
        if (s->last_kind) {
            s->last_kind[i] = 4; s->last_source[i] = -1; s->last_dest[i] = -1;
            s->last_mover[i] = (int8_t)mover;
        }
    } else {
        if (verify) {
            legal_cells(e, mover, scratch);
            if (action < 0 || action >= g->C || !scratch[action]) return ST_ILLEGAL;
        }
        int cell = (int)action;
        e->pc[cell] = 0; e->own[cell] = (int8_t)mover;            /* mechanics.py:463-479 */
        if (s->last_kind) {
            s->last_kind[i] = 0; s->last_source[i] = -1; s->last_dest[i] = (int16_t)cell;
            s->last_mover[i] = (int8_t)mover;
            s->last_dest_by_player[i * 2 + mover] = (int16_t)cell;
        }
        if (s->comp_labels) place_update(e, cell);
    }
    if (s->pass_streak) {
        if (is_pass) { s->pass_streak[i] += 1; s->pass_flags[i * 2 + mover] = 1; }
        else { s->pass_streak[i] = 0; s->pass_flags[i * 2 + mover] = 0; }
    }
    if (!is_pass && g->effect[phase] == EFF_REVERSI) {             /* effects.py:50-102 */
        int16_t mark[64];
        int m = custodial_from(e, s->last_dest[i], mover, 0, mark);
        for (int k = 0; k < m; k++) if (e->own[mark[k]] >= 0) e->own[mark[k]] = (int8_t)mover;
        s->scores[i * 2 + mover] = count_owned(e, mover);
        s->scores[i * 2 + (1 - mover)] = count_owned(e, 1 - mover);
    } else if (!is_pass && g->effect[phase] == EFF_PENTE) {        /* effects.py:29-48 */
        int16_t mark[64];
        int m = custodial_from(e, s->last_dest[i], mover, 2, mark);
        int gained = 0;
        for (int k = 0; k < m; k++)
            if (e->own[mark[k]] >= 0) { gained++; e->own[mark[k]] = -1; e->pc[mark[k]] = -1; }
        s->scores[i * 2 + mover] += gained;
    }
    if (s->scores) {
        if (s->scores[i * 2] < 0) s->scores[i * 2] = 0;
        if (s->scores[i * 2 + 1] < 0) s->scores[i * 2 + 1] = 0;
    }
    /* advancement (compiler.py:528-539) */
    int nxt = pos + 1, next_phase = phase, next_pos = nxt;
    if (nxt >= g->olen[phase]) { next_pos = 0; if (g->once[phase]) next_phase = phase + 1; }
    int next_player = next_phase < g->nphase ? g->order[next_phase][next_pos] : 0;
    /* end rules in order, first firing wins (compiler.py:563-573) */
    for (int r = 0; r < g->nend; r++) {
        int fired = 0;
        switch (g->end_kind[r]) {
        case END_LINE: fired = line_sat(e, mover, g->end_anch[r], g->end_arg[r]); break;
        case END_LINE_LOSE: fired = line_sat(e, mover, g->end_anch[r], g->end_arg[r]); break;
        case END_FULL: { fired = 1; for (int c = 0; c < g->C; c++) if (e->own[c] < 0) { fired = 0; break; } } break;
        case END_CONN: fired = mover == g->end_gate[r] && connected2(e, mover, g->end_ea[r], g->end_eb[r]); break;
        case END_PASSED_BOTH: fired = s->pass_streak[i] >= 2; break;
        case END_SCORE_GE: fired = s->scores[i * 2 + mover] >= g->end_arg[r]; break;
        }
        if (fired) {
            int8_t out = 0;
            if (g->end_res[r] == RES_MOVER_WIN) out = (int8_t)(1 + mover);
            else if (g->end_res[r] == RES_MOVER_LOSE) out = (int8_t)(2 - mover);
            else if (g->end_res[r] == RES_BY_SCORE) {      /* compiler.py:586-591 */
                int a = s->scores[i * 2], b = s->scores[i * 2 + 1];
                out = a > b ? 1 : (b > a ? 2 : 0);
            }
            s->outcome[i] = out;
            s->terminated[i] = 1;
            break;
        }
    }
    s->move_count[i] += 1;
    s->current_player[i] = (int8_t)next_player;
    if (s->phase) s->phase[i] = (int8_t)next_phase;
    return ST_OK;
}

/* --- movement / gridworld (mechanics.py:44-404, 518-608) --------------------- */

static inline int must_of(const env_t *e) { return e->s->must_move ? e->s->must_move[e->i] : -1; }

/* MovementMechanics._src_ok (mechanics.py:116-126) */
static inline int mv_src_ok(const env_t *e, int mover, int piece, int c, int use_must) {
    if (e->pc[c] != piece || e->own[c] != mover) return 0;
    if (use_must && e->g->L_must) { int mm = must_of(e); if (mm >= 0 && c != mm) return 0; }
    return 1;
}

static inline int mv_over_ok(const env_t *e, int gi, int mover, int mid) {
    const orc_game *g = e->g;
    if (mid == g->C) return 0;
    int mo = e->own[mid];
    if (mo < 0) return 0;
    if (g->grp[gi].over == OVER_OPP && mo != 1 - mover) return 0;
    if (g->grp[gi].over == OVER_MOVER && mo != mover) return 0;
    return 1;
}

/* per-source legal counts of one group (MovementMechanics.compute,
   mechanics.py:134-187); returns the group total */
static int mv_group_counts(const env_t *e, int gi, int mover, int16_t *cnt) {
    const orc_game *g = e->g;
    int C = g->C, d = g->grp[gi].d[mover], total = 0;
    for (int c = 0; c < C; c++) {
        int n = 0;
        if (mv_src_ok(e, mover, g->grp[gi].piece, c, 1)) {
            if (g->grp[gi].kind == K_STEP) {
                int x = g->nbr[d][c];
                n = x != C && e->own[x] < 0;
            } else if (g->grp[gi].kind == K_HOP) {
                int mid = g->nbr[d][c], two = mid != C ? g->nbr[d][mid] : C;
                n = mv_over_ok(e, gi, mover, mid) && two != C && e->own[two] < 0;
            } else {
                int x = g->nbr[d][c];
                for (int k = 0; k < g->grp[gi].L && x != C && e->own[x] < 0; k++) { n++; x = g->nbr[d][x]; }
            }
        }
        if (cnt) cnt[c] = (int16_t)n;
        total += n;
    }
    return total;
}

/* group totals with move priority (mechanics.py:188-197); returns the sum */
static int mv_compute(const env_t *e, int mover, int *tot) {
    const orc_game *g = e->g;
    int minp = 1000000, n = 0;
    for (int gi = 0; gi < g->ng; gi++) {
        tot[gi] = mv_group_counts(e, gi, mover, NULL);
        if (tot[gi] > 0 && g->grp[gi].prio < minp) minp = g->grp[gi].prio;
    }
    for (int gi = 0; gi < g->ng; gi++) {
        if (g->multi_prio && g->grp[gi].prio != minp) tot[gi] = 0;
        n += tot[gi];
    }
    return n;
}

static int mv_dest(const orc_game *g, int gi, int mover, int src, int k) {
    int d = g->grp[gi].d[mover], x = g->nbr[d][src];
    if (g->grp[gi].kind == K_HOP) return g->nbr[d][x];
    for (int j = 0; j < k; j++) x = g->nbr[d][x];      /* slide: k-th reach cell */
    return x;
}

/* GridworldMechanics (mechanics.py:529-548): the walker is the first cell
   holding the mover's walker (argmax -> 0 when none) */
static int gw_src(const env_t *e, int mover) {
    for (int c = 0; c < e->g->C; c++)
        if (e->pc[c] == e->g->grid_piece && e->own[c] == mover) return c;
    return 0;
}
static int gw_compute(const env_t *e, int mover, int *ok) {
    const orc_game *g = e->g;
    int src = gw_src(e, mover), n = 0;
    for (int k = 0; k < g->grid_ndir; k++) {
        int x = g->nbr[g->grid_dir[k]][src];
        ok[k] = x != g->C && e->own[x] < 0;
        n += ok[k];
    }
    return n;
}

/* number of legal actions of `mover` (without pass) */
static int mv_count(const env_t *e, int mover) {
    int tot[MAXG];
    return e->g->mech == MECH_GRID ? gw_compute(e, mover, tot) : mv_compute(e, mover, tot);
}

/* legal mask row (full_mask, mechanics.py:234-266 / 564-568) */
static void mv_mask(const env_t *e, int mover, uint8_t *row) {
    const orc_game *g = e->g;
    int tot[MAXG];
    memset(row, 0, g->A);
    if (g->mech == MECH_GRID) { gw_compute(e, mover, tot); for (int k = 0; k < g->grid_ndir; k++) row[k] = tot[k]; return; }
    mv_compute(e, mover, tot);
    int16_t cnt[MAXC];
    for (int gi = 0; gi < g->ng; gi++) {
        if (!tot[gi]) continue;
        mv_group_counts(e, gi, mover, cnt);
        for (int c = 0; c < g->C; c++)
            for (int k = 0; k < cnt[c]; k++)
                row[c * g->C + mv_dest(g, gi, mover, c, k)] = 1;
    }
}

/* MovementMechanics.sample (mechanics.py:199-232) */
static int64_t mv_sample(const env_t *e, int mover, double u) {
    const orc_game *g = e->g;
    int tot[MAXG];
    int n = g->mech == MECH_GRID ? gw_compute(e, mover, tot) : mv_compute(e, mover, tot);
    if (n == 0) return -1;
    int64_t r = (int64_t)(u * (double)n);
    if (r > n - 1) r = n - 1;
    int ng = g->mech == MECH_GRID ? g->grid_ndir : g->ng;
    for (int gi = 0; gi < ng; gi++) {
        if (r >= tot[gi]) { r -= tot[gi]; continue; }
        if (g->mech == MECH_GRID) return gi;
        int16_t cnt[MAXC];
        mv_group_counts(e, gi, mover, cnt);
        for (int c = 0; c < g->C; c++) {
            if (r < cnt[c]) return (int64_t)c * g->C + mv_dest(g, gi, mover, c, (int)r);
            r -= cnt[c];
        }
    }
    return -1;
}

/* first group claiming (src, dst) (MovementMechanics.apply, mechanics.py:283-322) */
static int mv_claim(const env_t *e, int mover, int src, int dst) {
    const orc_game *g = e->g;
    int C = g->C;
    for (int gi = 0; gi < g->ng; gi++) {
        if (!mv_src_ok(e, mover, g->grp[gi].piece, src, 1)) continue;
        int d = g->grp[gi].d[mover], match = 0;
        if (g->grp[gi].kind == K_STEP) {
            match = g->nbr[d][src] == dst && e->own[dst] < 0;
        } else if (g->grp[gi].kind == K_HOP) {
            int mid = g->nbr[d][src], two = mid != C ? g->nbr[d][mid] : C;
            match = two == dst && mv_over_ok(e, gi, mover, mid) && e->own[dst] < 0;
        } else {
            int pos = g->nbr[d][src], clear = 1;
            for (int k = 0; k < g->grp[gi].L; k++) {
                clear = clear && pos != C && e->own[pos] < 0;
                if (clear && pos == dst) match = 1;
                pos = pos != C ? g->nbr[d][pos] : C;
            }
        }
        if (match) return gi;
    }
    return -1;
}

static int mv_legal_action(const env_t *e, int mover, int64_t a) {
    const orc_game *g = e->g;
    if (g->mech == MECH_GRID) {
        int ok[8];
        gw_compute(e, mover, ok);
        return a >= 0 && a < g->grid_ndir && ok[a];
    }
    if (a < 0 || a >= (int64_t)g->C * g->C) return 0;
    int gi = mv_claim(e, mover, (int)(a / g->C), (int)(a % g->C));
    if (gi < 0) return 0;
    if (g->multi_prio) {                               /* mechanics.py:329-338 */
        int minp = 1000000;
        for (int k = 0; k < g->ng; k++)
            if (mv_group_counts(e, k, mover, NULL) > 0 && g->grp[k].prio < minp) minp = g->grp[k].prio;
        if (g->grp[gi].prio > minp) return 0;
    }
    return 1;
}

/* MovementMechanics.can_move_again (mechanics.py:368-403) */
static int mv_can_move_again(const env_t *e, int mover, int kind) {
    const orc_game *g = e->g;
    orc_soa *s = e->s;
    int ld = s->last_dest[e->i];
    if (!(ld >= 0 && s->last_mover[e->i] == mover)) return 0;
    for (int gi = 0; gi < g->ng; gi++) {
        if (g->grp[gi].kind != kind) continue;
        if (!mv_src_ok(e, mover, g->grp[gi].piece, ld, 0)) continue;
        int d = g->grp[gi].d[mover], x = g->nbr[d][ld];
        if (kind == K_HOP) {
            int two = x != g->C ? g->nbr[d][x] : g->C;
            if (mv_over_ok(e, gi, mover, x) && two != g->C && e->own[two] < 0) return 1;
        } else if (x != g->C && e->own[x] < 0) {
            return 1;
        }
    }
    return 0;
}

static inline void set_last(orc_soa *s, int64_t i, int kind, int src, int dst, int mover) {
    if (!s->last_kind) return;
    s->last_kind[i] = (int8_t)kind; s->last_source[i] = (int16_t)src; s->last_dest[i] = (int16_t)dst;
    s->last_mover[i] = (int8_t)mover; s->last_dest_by_player[i * 2 + mover] = (int16_t)dst;
}

/* CompiledGame.step_into for one live row of a movement / gridworld game
   (compiler.py:456-580) */
static void mv_step_one(env_t *e, int64_t action) {
    const orc_game *g = e->g;
    orc_soa *s = e->s;
    int64_t i = e->i;
    int C = g->C, mover = s->current_player[i];
    int ovr = -1, samep = 0;
    if (g->mech == MECH_GRID) {                        /* mechanics.py:570-602 */
        int src = gw_src(e, mover), ok[8];
        gw_compute(e, mover, ok);
        if (action >= 0 && action < g->grid_ndir && ok[action]) {
            int dst = g->nbr[g->grid_dir[action]][src];
            e->pc[dst] = (int8_t)g->grid_piece; e->own[dst] = (int8_t)mover;
            e->pc[src] = -1; e->own[src] = -1;
            set_last(s, i, K_STEP, src, dst, mover);
        }
    } else {
        int src = (int)(action / C), dst = (int)(action % C);
        int gi = mv_claim(e, mover, src, dst);
        if (gi >= 0) {
            int8_t pv = e->pc[src], ov = e->own[src];
            e->pc[src] = -1; e->own[src] = -1;
            e->pc[dst] = pv; e->own[dst] = ov;
            if (g->grp[gi].kind == K_HOP && g->grp[gi].capture) {
                int mid = g->nbr[g->grp[gi].d[mover]][src];
                e->pc[mid] = -1; e->own[mid] = -1;
            }
            set_last(s, i, g->grp[gi].kind, src, dst, mover);
        }
        /* effects in order (effects.py) */
        if (g->promote) {                              /* (promote pawn king (edge forward)) */
            int edge = mover == 0 ? 0 : 1;             /* P1 forward up -> top, P2 down -> bottom */
            for (int c = 0; c < C; c++)
                if (g->edge[edge][c] && e->pc[c] == g->promote_from && e->own[c] == mover)
                    e->pc[c] = (int8_t)g->promote_to;
        }
        if (g->extra_hop) {
            if (s->last_mover[i] == mover && s->last_kind[i] == K_HOP && mv_can_move_again(e, mover, K_HOP)) {
                ovr = mover; samep = 1;
            }
        }
        if (g->cap_custodial) {                        /* anchored custodial, any length */
            int16_t mark[64];
            int ld = s->last_dest[i];
            int m = (ld >= 0 && s->last_mover[i] == mover) ? custodial_from(e, ld, mover, 0, mark) : 0;
            for (int k = 0; k < m; k++) if (e->own[mark[k]] >= 0) { e->own[mark[k]] = -1; e->pc[mark[k]] = -1; }
        }
        if (g->corner_cust) {                          /* exprs.py:381-408, anchored */
            int ld = s->last_dest[i], hit[4];
            for (int k = 0; k < g->ncorner; k++) {
                int c = g->corner[k][0], n1 = g->corner[k][1], n2 = g->corner[k][2];
                hit[k] = e->own[c] == 1 - mover && e->pc[c] == 0 && e->own[n1] == mover && e->own[n2] == mover
                         && (ld == n1 || ld == n2) && s->last_mover[i] == mover;
            }
            for (int k = 0; k < g->ncorner; k++)
                if (hit[k]) { int c = g->corner[k][0]; e->own[c] = -1; e->pc[c] = -1; }
        }
    }
    /* advancement + extra-turn override + must_move (compiler.py:528-545) */
    int phase = phase_of(e), pos = 0;
    for (int k = 0; k < g->olen[phase]; k++) if (g->order[phase][k] == mover) { pos = k; break; }
    int nxt = pos + 1, next_phase = phase, next_pos = nxt;
    if (nxt >= g->olen[phase]) { next_pos = 0; if (g->once[phase]) next_phase = phase + 1; }
    int next_player = next_phase < g->nphase ? g->order[next_phase][next_pos] : 0;
    if (ovr >= 0) { next_player = ovr; next_phase = phase; }
    if (s->must_move) s->must_move[i] = (int16_t)((ovr >= 0 && samep) ? s->last_dest[i] : -1);
    int next_count = 0;
    if (g->needs_next) next_count = mv_count(e, next_player);
    for (int r = 0; r < g->nend; r++) {
        int fired = 0;
        switch (g->end_kind[r]) {
        case END_NO_LEGAL: fired = next_count == 0; break;
        case END_LAST_MOVE_IN: {
            int ld = s->last_dest[i];
            fired = (g->end_gate[r] < 0 || mover == g->end_gate[r]) && ld >= 0
                    && s->last_mover[i] == mover && g->end_mask[r][ld];
        } break;
        case END_LINE_EXCL: {                          /* global line, exprs.py:433-450 */
            if (mover != g->end_gate[r]) break;
            int t = g->end_arg[r];
            for (int w = 0; w < g->lt[t].nwin && !fired; w++) {
                int ok = 1;
                for (int j = 0; j < g->lt[t].len && ok; j++) {
                    int c = g->lt[t].win[w][j];
                    ok = e->own[c] == mover && e->pc[c] == 0 && !g->end_mask[r][c];
                }
                fired = ok;
            }
        } break;
        }
        if (fired) {
            s->outcome[i] = (int8_t)(g->end_res[r] == RES_MOVER_WIN ? 1 + mover : 2 - mover);
            s->terminated[i] = 1;
            break;
        }
    }
    s->move_count[i] += 1;
    s->current_player[i] = (int8_t)next_player;
    if (s->phase) s->phase[i] = (int8_t)next_phase;
}

/* --- exported API ----------------------------------------------------------- */

/* CompiledGame.init (compiler.py:329-364): start template broadcast + seeds */
void orc_init(const orc_game *g, orc_soa *s, int64_t B, const uint64_t *seeds) {
    for (int64_t i = 0; i < B; i++) {
        env_t e = env_of(g, s, i);
        memset(e.own, -1, g->C); memset(e.pc, -1, g->C);
        s->current_player[i] = (int8_t)g->order[0][0];
        s->move_count[i] = 0; s->terminated[i] = 0; s->truncated[i] = 0; s->outcome[i] = -1;
        s->seeds[i] = seeds[i];
        if (s->scores) { s->scores[2 * i] = 0; s->scores[2 * i + 1] = 0; }
        if (s->pass_streak) { s->pass_streak[i] = 0; s->pass_flags[2 * i] = 0; s->pass_flags[2 * i + 1] = 0; }
        if (s->last_kind) {
            s->last_mover[i] = -1; s->last_kind[i] = -1; s->last_source[i] = -1; s->last_dest[i] = -1;
            s->last_dest_by_player[2 * i] = -1; s->last_dest_by_player[2 * i + 1] = -1;
        }
        if (s->comp_labels) for (int c = 0; c < g->C; c++) s->comp_labels[i * g->C + c] = -1;
        if (s->phase) s->phase[i] = 0;
        if (s->must_move) s->must_move[i] = -1;
        for (int k = 0; k < g->nstart; k++) {
            e.own[g->start_cell[k]] = (int8_t)g->start_player[k];
            e.pc[g->start_cell[k]] = (int8_t)g->start_piece[k];
        }
        if (g->game == 3) {                                    /* reversi.ldx start */
            e.own[28] = 0; e.own[35] = 0; e.own[27] = 1; e.own[36] = 1;
            e.pc[28] = e.pc[35] = e.pc[27] = e.pc[36] = 0;
            s->scores[2 * i] = 2; s->scores[2 * i + 1] = 2;
        }
    }
}

void orc_spawn_seeds(uint64_t seed, int64_t first, int64_t B, uint64_t *out) {   /* rng.py:52-54 */
    for (int64_t i = 0; i < B; i++) out[i] = hash2(seed, (uint64_t)(first + i));
}

uint64_t orc_hash_key3(uint64_t a, uint64_t b, uint64_t c) {
    return mix64(mix64(mix64(0x243F6A8885A308D3ull ^ a) ^ b) ^ c);
}

void orc_legal(const orc_game *g, orc_soa *s, int64_t B, uint8_t *mask, int64_t *counts) {
    uint8_t cells[MAXC];
    for (int64_t i = 0; i < B; i++) {
        env_t e = env_of(g, s, i);
        if (g->mech != MECH_PLACE) {
            int term = s->terminated[i];
            if (mask) { if (term) memset(mask + i * g->A, 0, g->A); else mv_mask(&e, s->current_player[i], mask + i * g->A); }
            if (counts) counts[i] = term ? 0 : mv_count(&e, s->current_player[i]);
            continue;
        }
        int64_t t = legal_count_and_mask(&e, cells, mask ? mask + i * g->A : NULL);
        if (counts) counts[i] = t;
    }
}

void orc_sample(const orc_game *g, orc_soa *s, int64_t B, const double *u, int64_t *actions) {
    uint8_t cells[MAXC];
    for (int64_t i = 0; i < B; i++) {
        env_t e = env_of(g, s, i);
        double ui = u ? u[i] : uniform2(s->seeds[i], (uint64_t)s->move_count[i]);
        if (g->mech != MECH_PLACE) { actions[i] = s->terminated[i] ? -1 : mv_sample(&e, s->current_player[i], ui); continue; }
        actions[i] = sample_one(&e, ui, cells);
    }
}

/* rows may be NULL (all rows); returns status and the first bad row */
int orc_step(const orc_game *g, orc_soa *s, int64_t B, const int64_t *actions,
             const uint8_t *rows, int verify, int64_t *bad_row) {
    uint8_t cells[MAXC];
    if (verify) {
        /* verification happens before any mutation in the reference */
        for (int64_t i = 0; i < B; i++) {
            if (s->terminated[i] || (rows && !rows[i])) continue;
            env_t e = env_of(g, s, i);
            int mover = s->current_player[i], p = phase_of(&e);
            int64_t a = actions[i];
            if (g->mech != MECH_PLACE) {
                if (!mv_legal_action(&e, mover, a)) { if (bad_row) *bad_row = i; return ST_ILLEGAL; }
                continue;
            }
            int n = legal_cells(&e, mover, cells);
            int ok = (g->has_pass && a == g->pass_index) ? (n == 0 && g->force_pass[p])
                                                          : (a >= 0 && a < g->C && cells[a]);
            if (!ok) { if (bad_row) *bad_row = i; return ST_ILLEGAL; }
        }
    }
    for (int64_t i = 0; i < B; i++) {
        if (s->terminated[i] || (rows && !rows[i])) continue;
        env_t e = env_of(g, s, i);
        if (g->mech != MECH_PLACE) mv_step_one(&e, actions[i]);
        else step_one(&e, actions[i], 0, cells);
    }
    return ST_OK;
}

/* engine.playout_random (engine.py:123-163) for rows [lo, hi) */
static int64_t playout_range(const orc_game *g, orc_soa *s, int64_t lo, int64_t hi,
                             int max_turns, int64_t *stuck_row) {
    uint8_t cells[MAXC];
    int64_t steps = 0;
    for (int64_t i = lo; i < hi; i++) {
        env_t e = env_of(g, s, i);
        while (!s->terminated[i] && s->move_count[i] < max_turns) {
            double u = uniform2(s->seeds[i], (uint64_t)s->move_count[i]);
            int64_t a = g->mech != MECH_PLACE ? mv_sample(&e, s->current_player[i], u)
                                              : sample_one(&e, u, cells);
            if (a < 0) { if (stuck_row && *stuck_row < 0) *stuck_row = i; break; }
            if (g->mech != MECH_PLACE) mv_step_one(&e, a);
            else step_one(&e, a, 0, cells);
            steps++;
        }
        if (!s->terminated[i]) { s->terminated[i] = 1; s->truncated[i] = 1; s->outcome[i] = 0; }
    }
    return steps;
}

typedef struct { const orc_game *g; orc_soa *s; int64_t lo, hi; int max_turns; int64_t steps, stuck; } job_t;

static void *job_run(void *p) {
    job_t *j = (job_t *)p;
    j->stuck = -1;
    j->steps = playout_range(j->g, j->s, j->lo, j->hi, j->max_turns, &j->stuck);
    return NULL;
}

/* returns total env steps; *stuck_row = first row with no legal action (-1 if none) */
int64_t orc_playout(const orc_game *g, orc_soa *s, int64_t B, int max_turns, int nthreads,
                    int64_t *stuck_row) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    job_t jobs[256];
    pthread_t th[256];
    int64_t chunk = (B + nthreads - 1) / nthreads, total = 0;
    for (int t = 0; t < nthreads; t++) {
        jobs[t].g = g; jobs[t].s = s; jobs[t].max_turns = max_turns;
        jobs[t].lo = t * chunk < B ? t * chunk : B;
        jobs[t].hi = (t + 1) * chunk < B ? (t + 1) * chunk : B;
        pthread_create(&th[t], NULL, job_run, &jobs[t]);
    }
    if (stuck_row) *stuck_row = -1;
    for (int t = 0; t < nthreads; t++) {
        pthread_join(th[t], NULL);
        total += jobs[t].steps;
        if (stuck_row && jobs[t].stuck >= 0 && (*stuck_row < 0 || jobs[t].stuck < *stuck_row))
            *stuck_row = jobs[t].stuck;
    }
    return total;
}
