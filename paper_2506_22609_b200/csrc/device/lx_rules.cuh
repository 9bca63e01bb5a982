// lx_rules.cuh -- per-env rule templates shared by every kernel: the HBM
// word layout (pack/unpack), start position, sampling and the ply itself.
// Host-compilable on purpose (no CUDA builtins beyond lx_core.cuh), so the
// CPU test suite can run the generated rules through tests/hostsim.
//
// G::MECH selects the mechanic family of the lowered game:
//   0 placement  -- G::legal(s) is the bitboard of legal cells
//   1 movement   -- G::count_moves / select_move / move_legal / apply_move
//   2 gridworld  -- same interface, actions are direction indices
#pragma once

namespace lx {

// HBM word layout of one env (compact, per game): the boards and private
// words, the 64-bit seed, the two int32 scores when the game keeps scores,
// then bit fields holding only the meta the game's rules and the reference
// StateLayout need (state.py:34-66): move_count (32 bits), current player,
// terminated, truncated, outcome (+1), then, when present, phase, turn
// position, pass streak (int16) + pass flags, the last action (mover +1,
// kind +1, dest / per-player dests / source as cell index + 1) and
// must_move (cell + 1).  Connect Four packs into 32 B (NQ = 2) instead of 48.
__host__ __device__ constexpr int bitlen(int v) { return v <= 0 ? 0 : 1 + bitlen(v >> 1); }

template <class G>
struct Layout {
    static constexpr int W = G::W, NX = G::NX;
    static constexpr int SEED = 2 * W + NX;                      // seed lo, hi
    static constexpr int SCORE = SEED + 2;                       // sc0, sc1 (int32)
    static constexpr int CB = bitlen(G::C);                      // cell index + 1
    static constexpr int O_MC = 32 * (SCORE + (G::L_SCORES ? 2 : 0));
    static constexpr int O_CUR = O_MC + 32;
    static constexpr int O_TERM = O_CUR + 1, O_TRUNC = O_TERM + 1, O_OUT = O_TRUNC + 1;
    static constexpr int B_PHASE = G::L_PHASE ? bitlen(G::NPHASE) : 0;
    static constexpr int O_PHASE = O_OUT + 2;
    static constexpr int B_POS = G::L_TURNPOS ? 5 : 0;
    static constexpr int O_POS = O_PHASE + B_PHASE;
    static constexpr int B_PASS = G::L_PASSING ? 16 : 0;
    static constexpr int O_PASS = O_POS + B_POS;
    static constexpr int O_PF = O_PASS + B_PASS;                 // pf0, pf1
    static constexpr int B_LAST = G::L_LAST ? CB : 0;
    static constexpr int O_LM = O_PF + (G::L_PASSING ? 2 : 0);   // last_mover + 1 (2 bits)
    static constexpr int O_LK = O_LM + (G::L_LAST ? 2 : 0);      // last_kind + 1 (3 bits)
    static constexpr int O_LD = O_LK + (G::L_LAST ? 3 : 0);      // last_dest + 1
    static constexpr int O_L0 = O_LD + B_LAST;                   // ldbp0 + 1
    static constexpr int O_L1 = O_L0 + B_LAST;                   // ldbp1 + 1
    static constexpr int B_SRC = (G::L_LAST && G::MECH != 0) ? CB : 0;
    static constexpr int O_SRC = O_L1 + B_LAST;                  // last_source + 1
    static constexpr int B_MUST = G::L_MUSTMOVE ? CB : 0;
    static constexpr int O_MUST = O_SRC + B_SRC;                 // must_move + 1
    static constexpr int END = O_MUST + B_MUST;
    static constexpr int NWORDS = (END + 31) / 32;
    static constexpr int NQ = (NWORDS + 3) / 4;
};

// bit field [OFF, OFF + BITS) of a word array (BITS <= 32)
template <int OFF, int BITS>
__device__ __forceinline__ u32 getf(const u32* w) {
    constexpr int wi = OFF >> 5, sh = OFF & 31;
    constexpr u32 mask = BITS >= 32 ? 0xffffffffu : ((1u << BITS) - 1u);
    if constexpr (BITS == 0) {
        return 0u;
    } else if constexpr (sh + BITS <= 32) {
        return (w[wi] >> sh) & mask;
    } else {
        return ((w[wi] >> sh) | (w[wi + 1] << (32 - sh))) & mask;
    }
}
// OR v into the field (the word array starts zeroed)
template <int OFF, int BITS>
__device__ __forceinline__ void putf(u32* w, u32 v) {
    constexpr int wi = OFF >> 5, sh = OFF & 31;
    constexpr u32 mask = BITS >= 32 ? 0xffffffffu : ((1u << BITS) - 1u);
    if constexpr (BITS > 0) {
        v &= mask;
        w[wi] |= v << sh;
        if constexpr (sh + BITS > 32) w[wi + 1] |= v >> (32 - sh);
    }
}

template <class G>
__device__ __forceinline__ void unpack(typename G::St& s, const u32 (&w)[Layout<G>::NQ * 4]) {
    typedef Layout<G> L;
    constexpr int W = G::W;
#pragma unroll
    for (int i = 0; i < W; i++) { s.own0.w[i] = w[i]; s.own1.w[i] = w[W + i]; }
#pragma unroll
    for (int i = 0; i < G::NX; i++) s.ext[i] = w[2 * W + i];
    s.seed = (u64)w[L::SEED] | ((u64)w[L::SEED + 1] << 32);
    s.sc0 = G::L_SCORES ? (int)w[L::SCORE] : 0;
    s.sc1 = G::L_SCORES ? (int)w[L::SCORE + 1] : 0;
    s.mc = getf<L::O_MC, 32>(w);
    s.cur = (int)getf<L::O_CUR, 1>(w);
    s.term = (int)getf<L::O_TERM, 1>(w);
    s.trunc = (int)getf<L::O_TRUNC, 1>(w);
    s.outcome = (int)getf<L::O_OUT, 2>(w) - 1;
    s.phase = (int)getf<L::O_PHASE, L::B_PHASE>(w);
    s.pos = (int)getf<L::O_POS, L::B_POS>(w);
    s.pass_streak = G::L_PASSING ? (int)(short)getf<L::O_PASS, 16>(w) : 0;
    s.pf0 = G::L_PASSING ? (int)getf<L::O_PF, 1>(w) : 0;
    s.pf1 = G::L_PASSING ? (int)getf<L::O_PF + 1, 1>(w) : 0;
    if (G::L_LAST) {
        s.last_mover = (int)getf<L::O_LM, 2>(w) - 1;
        s.last_kind = (int)getf<L::O_LK, 3>(w) - 1;
        s.last_dest = (int)getf<L::O_LD, L::B_LAST>(w) - 1;
        s.ldbp0 = (int)getf<L::O_L0, L::B_LAST>(w) - 1;
        s.ldbp1 = (int)getf<L::O_L1, L::B_LAST>(w) - 1;
    } else {
        s.last_mover = -1; s.last_kind = -1; s.last_dest = -1; s.ldbp0 = -1; s.ldbp1 = -1;
    }
    s.last_source = L::B_SRC ? (int)getf<L::O_SRC, L::B_SRC>(w) - 1 : -1;
    s.must_move = L::B_MUST ? (int)getf<L::O_MUST, L::B_MUST>(w) - 1 : -1;
    s.ovr = -1;
    s.samep = 0;
    s.ncached = 0;
    s.mirror_fresh = 0;
    s.mirror_valid = 0;
}

template <class G>
__device__ __forceinline__ void pack(const typename G::St& s, u32 (&w)[Layout<G>::NQ * 4]) {
    typedef Layout<G> L;
    constexpr int W = G::W;
#pragma unroll
    for (int i = 2 * W + G::NX; i < L::NQ * 4; i++) w[i] = 0u;
#pragma unroll
    for (int i = 0; i < W; i++) { w[i] = s.own0.w[i]; w[W + i] = s.own1.w[i]; }
#pragma unroll
    for (int i = 0; i < G::NX; i++) w[2 * W + i] = s.ext[i];
    w[L::SEED] = (u32)s.seed;
    w[L::SEED + 1] = (u32)(s.seed >> 32);
    if (G::L_SCORES) { w[L::SCORE] = (u32)s.sc0; w[L::SCORE + 1] = (u32)s.sc1; }
    putf<L::O_MC, 32>(w, s.mc);
    putf<L::O_CUR, 1>(w, (u32)s.cur);
    putf<L::O_TERM, 1>(w, (u32)s.term);
    putf<L::O_TRUNC, 1>(w, (u32)s.trunc);
    putf<L::O_OUT, 2>(w, (u32)(s.outcome + 1));
    putf<L::O_PHASE, L::B_PHASE>(w, (u32)s.phase);
    putf<L::O_POS, L::B_POS>(w, (u32)s.pos);
    if (G::L_PASSING) {
        putf<L::O_PASS, 16>(w, (u32)s.pass_streak);
        putf<L::O_PF, 1>(w, (u32)s.pf0);
        putf<L::O_PF + 1, 1>(w, (u32)s.pf1);
    }
    if (G::L_LAST) {
        putf<L::O_LM, 2>(w, (u32)(s.last_mover + 1));
        putf<L::O_LK, 3>(w, (u32)(s.last_kind + 1));
        putf<L::O_LD, L::B_LAST>(w, (u32)(s.last_dest + 1));
        putf<L::O_L0, L::B_LAST>(w, (u32)(s.ldbp0 + 1));
        putf<L::O_L1, L::B_LAST>(w, (u32)(s.ldbp1 + 1));
    }
    putf<L::O_SRC, L::B_SRC>(w, (u32)(s.last_source + 1));
    putf<L::O_MUST, L::B_MUST>(w, (u32)(s.must_move + 1));
}

// start position (reference compiler.py:329-345 _build_template + init)
template <class G>
__device__ __forceinline__ void init_state(typename G::St& s, u64 seed) {
    s.own0 = bb_zero<G::W>();
    s.own1 = bb_zero<G::W>();
#pragma unroll
    for (int i = 0; i < (G::NX > 0 ? G::NX : 1); i++) s.ext[i] = 0u;
    s.mc = 0u;
    s.cur = G::FIRST_PLAYER;
    s.term = 0; s.trunc = 0; s.outcome = -1; s.phase = 0; s.pos = 0;
    s.last_mover = -1; s.last_kind = -1; s.last_dest = -1; s.last_source = -1;
    s.pass_streak = 0; s.pf0 = 0; s.pf1 = 0; s.ldbp0 = -1; s.ldbp1 = -1;
    s.sc0 = 0; s.sc1 = 0;
    s.must_move = -1; s.ovr = -1; s.samep = 0; s.ncached = 0; s.mirror_fresh = 0;
    s.mirror_valid = 0;
    s.seed = seed;
    G::start(s);
}

// number of legal non-pass actions for the current mover (reference
// CompiledGame.compute_all totals, compiler.py:379-392)
template <class G>
__device__ __forceinline__ int legal_count(const typename G::St& s) {
    if constexpr (G::MECH == 0) {
        return popc(G::legal(s));
    } else {
        int tot[G::NG];
        return G::count_moves(s, tot);
    }
}

// uniform legal action for the current mover; -1 when stuck
// (reference compiler.py:430-446, mechanics.py:209-242, 488-492).  `hint`
// receives the sampled move group (movement games) for apply_step.
#ifndef LX_EARLY_DRAW
#define LX_EARLY_DRAW 1
#endif
template <class G>
__device__ __forceinline__ int sample_action(const typename G::St& s, u64 smix, int& hint) {
    hint = -1;
    if constexpr (G::MECH == 0) {
#if LX_EARLY_DRAW
        // the uniform depends only on (seed, move_count): formed ahead of the
        // legality, in the same basic block, so the RNG / FP64 conversion
        // chain overlaps the bitboard work instead of following the count
        // (a shorter dependent chain per ply: latency-bound small batches, MCTS)
        const double u = key_uniform(mix64(smix ^ (u64)s.mc));
        const BB<G::W> legal = G::legal(s);
        const int n = popc(legal);
        if (n == 0) return G::force_pass(s.phase) ? G::PASS : -1;
        const int r = draw_index_u(u, n);
#else
        const BB<G::W> legal = G::legal(s);
        const int n = popc(legal);
        if (n == 0) return G::force_pass(s.phase) ? G::PASS : -1;
        const int r = draw_index(mix64(smix ^ (u64)s.mc), n);
#endif
        return G::bit_cell(select_bit(legal, r));
    } else {
        int tot[G::NG];
        int n = 0;
        if (s.ncached) {               // totals computed by the previous ply's lookahead
#pragma unroll
            for (int i = 0; i < G::NG; i++) { tot[i] = s.ntot[i]; n += tot[i]; }
        } else {
            n = G::count_moves(s, tot);
        }
        if (n == 0) return G::force_pass(s.phase) ? G::PASS : -1;
        const int r = draw_index(mix64(smix ^ (u64)s.mc), n);
        return G::select_move(s, r, tot, hint);
    }
}

template <class G>
__device__ __forceinline__ int sample_action(const typename G::St& s, u64 smix) {
    int hint;
    return sample_action<G>(s, smix, hint);
}

// one ply for a live row (reference compiler.py:456-580, order preserved:
// mechanic write, pass bookkeeping, effects, score clamp, advancement incl.
// extra-turn override and must_move, no_legal_actions lookahead, ordered end
// rules evaluated for the mover, counters).  Split in two around the
// mechanic write so lx_rollout can run a reach-set flood with the whole warp
// converged between them (apply_step_pre / apply_step_post).
template <class G>
__device__ __forceinline__ void ply_prologue(typename G::St& s) {
    s.ovr = -1;
    s.samep = 0;
    s.ncached = 0;
    s.mirror_fresh = 0;
    if constexpr (G::ROW_MIRROR) {          // first ply of this state in this kernel
        if (!s.mirror_valid) { G::rm_build(s); s.mirror_valid = 1; }
    }
    G::clear_transient(s);
}

template <class G>
__device__ __forceinline__ void ply_pass_write(typename G::St& s, int mover) {
    s.last_kind = 4; s.last_dest = -1; s.last_source = -1; s.last_mover = mover;
}

// everything after the mechanic write (mover / phase: the ply's, unchanged)
template <class G>
__device__ __forceinline__ void ply_tail(typename G::St& s, int action, bool is_pass, int mover,
                                         int phase) {
    if (G::L_PASSING) {
        if (is_pass) {
            s.pass_streak += 1;
            if (mover) s.pf1 = 1; else s.pf0 = 1;
        } else {
            s.pass_streak = 0;
            if (mover) s.pf1 = 0; else s.pf0 = 0;
        }
    }
    if (!is_pass) G::effects(s, action, mover, phase);
    if (G::L_SCORES) {
        s.sc0 = s.sc0 < 0 ? 0 : s.sc0;
        s.sc1 = s.sc1 < 0 ? 0 : s.sc1;
    }
    int next_player, next_phase, next_pos;
    G::advance(phase, s.pos, mover, next_player, next_phase, next_pos);
    if (s.ovr >= 0) { next_player = s.ovr; next_phase = phase; next_pos = s.pos; }   // extra turn
    if (G::L_MUSTMOVE) s.must_move = (s.ovr >= 0 && s.samep) ? s.last_dest : -1;
    int next_count = 0;
    if (G::NEEDS_NEXT_COUNT) {                                          // compiler.py:547-561
        typename G::St t = s;
        t.cur = next_player;
        t.phase = next_phase;
        if constexpr (G::MECH == 0) {
            next_count = legal_count<G>(t);
        } else {
            // the lookahead is exactly the next ply's legality: keep its group
            // totals for sample_action (the fused rollout stays in registers)
            next_count = G::count_moves(t, s.ntot);
            s.ncached = 1;
        }
        if (next_count == 0 && G::PASS >= 0 && G::force_pass(next_phase)) next_count = 1;
    }
    const int out = G::end_rules(s, mover, next_count);
    if (out >= 0) { s.term = 1; s.outcome = out; }
    s.mc += 1u;
    s.cur = next_player;
    s.phase = next_phase;
    if (G::L_TURNPOS) s.pos = next_pos;
}

template <class G>
__device__ __forceinline__ void apply_step(typename G::St& s, int action, int hint = -1) {
    const int mover = s.cur;
    const int phase = s.phase;
    const bool is_pass = (G::PASS >= 0) && action == G::PASS;
    ply_prologue<G>(s);
    if (is_pass) {
        ply_pass_write<G>(s, mover);
    } else {
        if constexpr (G::MECH == 0) {
            G::write_place(s, action, mover, phase);
        } else {
            G::apply_move(s, action, mover, hint);
        }
    }
    ply_tail<G>(s, action, is_pass, mover, phase);
}

// the first half of a placement ply up to the reach-set flood (G::SPLIT_FLOOD
// games): fl receives the flood's inputs (fl.need = 0: no flood)
template <class G>
__device__ __forceinline__ void apply_step_pre(typename G::St& s, int action,
                                               typename G::Flood& fl) {
    const int mover = s.cur;
    const int phase = s.phase;
    const bool is_pass = (G::PASS >= 0) && action == G::PASS;
    ply_prologue<G>(s);
    if (is_pass) {
        ply_pass_write<G>(s, mover);
        fl.need = 0;
    } else {
        G::write_place_pre(s, action, mover, phase, fl);
    }
}

// the rest of the ply once fl.f holds the flooded set
template <class G>
__device__ __forceinline__ void apply_step_post(typename G::St& s, int action,
                                                const typename G::Flood& fl) {
    const bool is_pass = (G::PASS >= 0) && action == G::PASS;
    if (!is_pass) G::flood_post(s, fl);
    ply_tail<G>(s, action, is_pass, s.cur, s.phase);
}

// legality of one action (reference mechanics.py:281-338, 499-512,
// compiler.py:484-494)
template <class G>
__device__ __forceinline__ bool action_legal(const typename G::St& s, i64 a) {
    if constexpr (G::MECH == 0) {
        const BB<G::W> legal = G::legal(s);
        if (G::PASS >= 0 && a == G::PASS) return !any(legal) && G::force_pass(s.phase);
        if (a < 0 || a >= G::C) return false;
        return test(legal, G::cell_bit((int)a));
    } else {
        if (G::PASS >= 0 && a == G::PASS) return legal_count<G>(s) == 0 && G::force_pass(s.phase);
        if (a < 0 || a >= (i64)(G::PASS >= 0 ? G::A - 1 : G::A)) return false;
        return G::move_legal(s, (int)a);
    }
}

}  // namespace lx
