/*
 * ludax_oracle.c -- CPU ORACLE FOR PARITY TESTS.  TEST INFRASTRUCTURE ONLY.
 *
 * A scalar, cell-array restatement of the reference's rollout hot path
 * (reference: /root/reference/pkg/src/boardlang/, the numpy "boardlang"
 * re-implementation of Ludax) for the five config games.  It works on the
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
enum { END_LINE = 0, END_FULL = 1, END_CONN = 2, END_PASSED_BOTH = 3, END_SCORE_GE = 4, END_LINE_LOSE = 5 };
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

static void build_custodial(orc_game *g) {
    static const char *axes[4] = {"right", "down", "down_right", "down_left"};
    static const char *inv[4] = {"left", "up", "up_left", "up_right"};
    g->ncust = 0;
    for (int a = 0; a < 4; a++) {
        g->cust_dir[g->ncust++] = dir_index_grid(axes[a]);
        g->cust_dir[g->ncust++] = dir_index_grid(inv[a]);
    }
    g->ray_max = 0;
    for (int i = 0; i < g->ncust; i++) {
        int l = ray_len(g, g->cust_dir[i]);
        if (l > g->ray_max) g->ray_max = l;
    }
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
/* layout bits: 1 scores, 2 passing, 4 last_action, 8 connectivity, 16 phase */
int orc_layout(const orc_game *g) {
    return g->L_scores | (g->L_passing << 1) | (g->L_last << 2) | (g->L_conn << 3) | (g->L_phase << 4);
}

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
        int64_t t = legal_count_and_mask(&e, cells, mask ? mask + i * g->A : NULL);
        if (counts) counts[i] = t;
    }
}

void orc_sample(const orc_game *g, orc_soa *s, int64_t B, const double *u, int64_t *actions) {
    uint8_t cells[MAXC];
    for (int64_t i = 0; i < B; i++) {
        env_t e = env_of(g, s, i);
        double ui = u ? u[i] : uniform2(s->seeds[i], (uint64_t)s->move_count[i]);
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
            int n = legal_cells(&e, mover, cells);
            int ok = (g->has_pass && a == g->pass_index) ? (n == 0 && g->force_pass[p])
                                                          : (a >= 0 && a < g->C && cells[a]);
            if (!ok) { if (bad_row) *bad_row = i; return ST_ILLEGAL; }
        }
    }
    for (int64_t i = 0; i < B; i++) {
        if (s->terminated[i] || (rows && !rows[i])) continue;
        env_t e = env_of(g, s, i);
        step_one(&e, actions[i], 0, cells);
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
            int64_t a = sample_one(&e, u, cells);
            if (a < 0) { if (stuck_row && *stuck_row < 0) *stuck_row = i; break; }
            step_one(&e, a, 0, cells);
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
