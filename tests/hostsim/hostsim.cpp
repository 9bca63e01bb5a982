// hostsim.cpp -- TEST INFRASTRUCTURE.  Runs a lowered game's rules on the CPU
// (same templates as the kernels: lx_core.cuh, lx_rules.cuh, generated
// struct Game) and exports the reference GameState layout, so the CPU test
// suite can compare the lowering against the oracle without a GPU.
// Built per game by tests/hostsim/hostsim.py with -DGAME_SOURCE="<file>".
#include "host_compat.h"
#include GAME_SOURCE          // its #defines (block shape, arena sizes) precede lx_core.cuh
#include "lx_rules.cuh"

#include <cstring>
#include <vector>

typedef Game::St St;

struct RefOut {
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
    int8_t *turn_pos;
    uint8_t *hopped_mask, *captured_mask, *promoted_mask;
};

static void export_one(const St& s, int64_t i, const RefOut* p) {
    for (int c = 0; c < Game::C; c++) {
        const int cb = Game::cell_bit(c);
        const bool a = lx::test(s.own0, cb), b = lx::test(s.own1, cb);
        p->board_owner[i * Game::C + c] = a ? 0 : (b ? 1 : -1);
        p->board_piece[i * Game::C + c] = (a || b) ? (int8_t)Game::piece_at(s, cb) : -1;
    }
    p->current_player[i] = (int8_t)s.cur;
    p->move_count[i] = (int32_t)s.mc;
    p->terminated[i] = (uint8_t)s.term;
    p->truncated[i] = (uint8_t)s.trunc;
    p->outcome[i] = (int8_t)s.outcome;
    p->seeds[i] = s.seed;
    if (p->scores) { p->scores[2 * i] = s.sc0; p->scores[2 * i + 1] = s.sc1; }
    if (p->pass_streak) {
        p->pass_streak[i] = (int16_t)s.pass_streak;
        p->pass_flags[2 * i] = (uint8_t)s.pf0;
        p->pass_flags[2 * i + 1] = (uint8_t)s.pf1;
    }
    if (p->last_mover) {
        p->last_mover[i] = (int8_t)s.last_mover;
        p->last_kind[i] = (int8_t)s.last_kind;
        p->last_source[i] = (int16_t)s.last_source;
        p->last_dest[i] = (int16_t)s.last_dest;
        p->last_dest_by_player[2 * i] = (int16_t)s.ldbp0;
        p->last_dest_by_player[2 * i + 1] = (int16_t)s.ldbp1;
    }
    if (p->comp_labels) Game::labels(s, (short*)(p->comp_labels + i * Game::CONN_PLANS * Game::C));
    if (p->phase) p->phase[i] = (int8_t)s.phase;
    if (p->must_move) p->must_move[i] = (int16_t)s.must_move;
    if (p->turn_pos) p->turn_pos[i] = (int8_t)s.pos;
    if (p->hopped_mask) Game::export_transient(s, p->hopped_mask + i * Game::C,
                                               p->captured_mask + i * Game::C,
                                               p->promoted_mask + i * Game::C);
}

// legal mask of the current mover (reference CompiledGame.legal_mask row)
static void mask_row(const St& s, uint8_t* row) {
    for (int a = 0; a < Game::A; a++) row[a] = 0;
    if (s.term) return;
    const int n = lx::legal_count<Game>(s);
    if constexpr (Game::MECH == 0) {
        lx::BB<Game::W> legal = Game::legal(s);
        for (int c = 0; c < Game::C; c++) row[c] = lx::test(legal, Game::cell_bit(c));
    } else {
        Game::enum_moves(s, [&](int a) { row[a] = 1; });
    }
    if (Game::PASS >= 0) row[Game::PASS] = n == 0 && Game::force_pass(s.phase);
}

// each game's .so keeps its own copies of the (identically named) inline
// rule functions and their static tables: built with -fvisibility=hidden
// -fno-gnu-unique, only these entry points are exported
#define SIM_API __attribute__((visibility("default")))

extern "C" {

// engine.playout_random from given seeds; also round-trips every state
// through pack/unpack each ply (checks the HBM word layout).
SIM_API int64_t sim_playout(int64_t B, const uint64_t* seeds, int max_turns, const RefOut* out) {
    int64_t steps = 0;
    for (int64_t i = 0; i < B; i++) {
        St s;
        lx::init_state<Game>(s, seeds[i]);
        const uint64_t smix = lx::seed_mix(s.seed);
        while (!s.term && (int)s.mc < max_turns) {
            int hint;
            const int a = lx::sample_action<Game>(s, smix, hint);
            if (a < 0) break;
            if constexpr (Game::SPLIT_FLOOD) {
                // the rollout's split ply: pre, the reach-set flood, post
                // (sim_masks / sim_transcript exercise the fused apply_step)
                Game::Flood fl;
                lx::apply_step_pre<Game>(s, a, fl);
                if (fl.need) {
                    typename Game::BBW g = (fl.f | Game::flood_dil_bb(fl.f)) & fl.free_;
                    while (!lx::equal(g, fl.f)) {
                        fl.f = g;
                        g = (fl.f | Game::flood_dil_bb(fl.f)) & fl.free_;
                    }
                }
                lx::apply_step_post<Game>(s, a, fl);
            } else {
                lx::apply_step<Game>(s, a, hint);
            }
            u32 w[lx::Layout<Game>::NQ * 4];
            lx::pack<Game>(s, w);
            lx::unpack<Game>(s, w);
            steps++;
        }
        if (!s.term) { s.term = 1; s.trunc = 1; s.outcome = 0; }
        export_one(s, i, out);
    }
    return steps;
}

// per-ply legal masks of env `seed` (A bytes per ply, up to max_plies)
SIM_API int sim_masks(uint64_t seed, int max_plies, uint8_t* masks, int64_t* actions) {
    St s;
    lx::init_state<Game>(s, seed);
    const uint64_t smix = lx::seed_mix(s.seed);
    int t = 0;
    for (; t < max_plies && !s.term; t++) {
        mask_row(s, masks + (int64_t)t * Game::A);
        int hint;
        const int a = lx::sample_action<Game>(s, smix, hint);
        actions[t] = a;
        if (a < 0) break;
        lx::apply_step<Game>(s, a, hint);
    }
    return t;
}

// scripted transcript from init(seed): per ply the mask before the move and
// whether the action was legal (verify path, no hint); stops at the first
// illegal action.  Exports the final state.  Returns plies applied.
SIM_API int sim_transcript(uint64_t seed, int n, const int64_t* actions, uint8_t* masks, uint8_t* legal,
                   const RefOut* out) {
    St s;
    lx::init_state<Game>(s, seed);
    int t = 0;
    for (; t < n && !s.term; t++) {
        mask_row(s, masks + (int64_t)t * Game::A);
        legal[t] = lx::action_legal<Game>(s, actions[t]);
        if (!legal[t]) break;
        lx::apply_step<Game>(s, (int)actions[t]);
    }
    mask_row(s, masks + (int64_t)t * Game::A);
    export_one(s, 0, out);
    return t;
}

}

// device state layout facts (lx::Layout), checked against the lowering's
// info["nwords"/"nq"] by the CPU suite
extern "C" SIM_API int sim_layout(int *out) {
    out[0] = lx::Layout<Game>::NWORDS;
    out[1] = lx::Layout<Game>::NQ;
    return 0;
}
