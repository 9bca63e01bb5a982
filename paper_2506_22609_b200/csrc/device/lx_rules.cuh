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

template <class G>
struct Layout {
    static constexpr int W = G::W, NX = G::NX;
    static constexpr int META = 2 * W + NX;
    static constexpr int NWORDS = META + 8;
    static constexpr int NQ = (NWORDS + 3) / 4;
};

template <class G>
__device__ __forceinline__ void unpack(typename G::St& s, const u32 (&w)[Layout<G>::NQ * 4]) {
    constexpr int W = G::W, M = Layout<G>::META;
#pragma unroll
    for (int i = 0; i < W; i++) { s.own0.w[i] = w[i]; s.own1.w[i] = w[W + i]; }
#pragma unroll
    for (int i = 0; i < G::NX; i++) s.ext[i] = w[2 * W + i];
    s.mc = w[M];
    const u32 f = w[M + 1];
    s.cur = f & 1u;
    s.term = (f >> 1) & 1u;
    s.trunc = (f >> 2) & 1u;
    s.outcome = (int)((f >> 3) & 3u) - 1;
    s.phase = (f >> 5) & 7u;
    s.last_mover = (int)((f >> 8) & 3u) - 1;
    s.pf0 = (f >> 10) & 1u;
    s.pf1 = (f >> 11) & 1u;
    s.last_kind = (int)((f >> 12) & 7u) - 1;
    s.pos = (f >> 15) & 31u;
    s.last_dest = (short)(w[M + 2] & 0xffffu);
    s.pass_streak = (short)(w[M + 2] >> 16);
    s.ldbp0 = (short)(w[M + 3] & 0xffffu);
    s.ldbp1 = (short)(w[M + 3] >> 16);
    s.sc0 = (short)(w[M + 4] & 0xffffu);
    s.sc1 = (short)(w[M + 4] >> 16);
    s.seed = (u64)w[M + 5] | ((u64)w[M + 6] << 32);
    s.last_source = (short)(w[M + 7] & 0xffffu);
    s.must_move = (short)(w[M + 7] >> 16);
    s.ovr = -1;
    s.samep = 0;
    s.ncached = 0;
}

template <class G>
__device__ __forceinline__ void pack(const typename G::St& s, u32 (&w)[Layout<G>::NQ * 4]) {
    constexpr int W = G::W, M = Layout<G>::META;
#pragma unroll
    for (int i = 0; i < W; i++) { w[i] = s.own0.w[i]; w[W + i] = s.own1.w[i]; }
#pragma unroll
    for (int i = 0; i < G::NX; i++) w[2 * W + i] = s.ext[i];
    w[M] = s.mc;
    w[M + 1] = (u32)s.cur | ((u32)s.term << 1) | ((u32)s.trunc << 2) |
               ((u32)(s.outcome + 1) << 3) | ((u32)s.phase << 5) |
               ((u32)(s.last_mover + 1) << 8) | ((u32)s.pf0 << 10) | ((u32)s.pf1 << 11) |
               ((u32)(s.last_kind + 1) << 12) | ((u32)s.pos << 15);
    w[M + 2] = ((u32)s.last_dest & 0xffffu) | ((u32)s.pass_streak << 16);
    w[M + 3] = ((u32)s.ldbp0 & 0xffffu) | ((u32)s.ldbp1 << 16);
    w[M + 4] = ((u32)s.sc0 & 0xffffu) | ((u32)s.sc1 << 16);
    w[M + 5] = (u32)s.seed;
    w[M + 6] = (u32)(s.seed >> 32);
    w[M + 7] = ((u32)s.last_source & 0xffffu) | ((u32)s.must_move << 16);
#pragma unroll
    for (int i = Layout<G>::NWORDS; i < Layout<G>::NQ * 4; i++) w[i] = 0u;
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
    s.must_move = -1; s.ovr = -1; s.samep = 0; s.ncached = 0;
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
template <class G>
__device__ __forceinline__ int sample_action(const typename G::St& s, u64 smix, int& hint) {
    hint = -1;
    if constexpr (G::MECH == 0) {
        const BB<G::W> legal = G::legal(s);
        const int n = popc(legal);
        if (n == 0) return G::force_pass(s.phase) ? G::PASS : -1;
        const int r = draw_index(mix64(smix ^ (u64)s.mc), n);
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
// rules evaluated for the mover, counters)
template <class G>
__device__ __forceinline__ void apply_step(typename G::St& s, int action, int hint = -1) {
    const int mover = s.cur;
    const int phase = s.phase;
    const bool is_pass = (G::PASS >= 0) && action == G::PASS;
    s.ovr = -1;
    s.samep = 0;
    s.ncached = 0;
    G::clear_transient(s);
    if (is_pass) {
        s.last_kind = 4; s.last_dest = -1; s.last_source = -1; s.last_mover = mover;
    } else {
        if constexpr (G::MECH == 0) {
            G::write_place(s, action, mover, phase);
        } else {
            G::apply_move(s, action, mover, hint);
        }
    }
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
