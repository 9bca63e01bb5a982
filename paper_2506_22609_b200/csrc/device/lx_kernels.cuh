// lx_kernels.cuh -- kernel templates instantiated once per game.
//
// Included at the end of every generated translation unit, after the
// lowering has defined `struct Game` (constants + rule device functions, see
// paper_2506_22609_b200/lowering.py).  All kernels are extern "C" so the
// native runtime finds them by name in the NVRTC cubin.
//
// HBM layout of a batch of B envs ("state words"): each env is NQ*4 32-bit
// words, stored quad-major -- quad q of env i lives at uint4 index q*B + i --
// so a warp moves 512 contiguous bytes per 128-bit load.  Word map:
//   [0, W)        P1 stones        [W, 2W)       P2 stones
//   [2W, 2W+NX)   piece-type planes (games with several piece types), then
//                 rule-private words (e.g. edge-connected stone sets)
//   then the seed, scores and packed meta bit fields (lx::Layout in
//   lx_rules.cuh), zero padding to NQ*4.
#pragma once

#include "lx_rules.cuh"

namespace lx {

__device__ __forceinline__ u64 globaltimer_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ u32 ld_acquire_gpu(const u32* p) {
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <class G>
__device__ __forceinline__ void load_state(typename G::St& s, const u32* __restrict__ st,
                                           i64 B, i64 i) {
    constexpr int NQ = Layout<G>::NQ;
    u32 w[NQ * 4];
    const uint4* q4 = reinterpret_cast<const uint4*>(st);
#pragma unroll
    for (int q = 0; q < NQ; q++) {
        const uint4 v = q4[(i64)q * B + i];
        w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
    unpack<G>(s, w);
}

template <class G>
__device__ __forceinline__ void store_state(const typename G::St& s, u32* __restrict__ st,
                                            i64 B, i64 i) {
    constexpr int NQ = Layout<G>::NQ;
    u32 w[NQ * 4];
    pack<G>(s, w);
    uint4* q4 = reinterpret_cast<uint4*>(st);
#pragma unroll
    for (int q = 0; q < NQ; q++)
        q4[(i64)q * B + i] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

__device__ __forceinline__ i64 gtid() { return (i64)blockIdx.x * blockDim.x + threadIdx.x; }

// 4 mask bits -> 4 bytes of 0/1
__device__ __forceinline__ u32 spread4(u32 x) { return ((x & 0xfu) * 0x00204081u) & 0x01010101u; }

// bool-mask rows of a full warp written from one concatenated bit stream
// (write_mask_rows; 0: the per-piece row walk, for A/B)
#ifndef LX_MASK_STREAM
#define LX_MASK_STREAM 1
#endif

// Stage the lane's legal-mask row as a bit vector in cell order (cells, then
// the pass column) in a per-warp shared-memory block of 32 rows x STRIDE
// words; returns the block.  Every lane of the warp must call it.
template <class G>
__device__ __forceinline__ const u32* stage_mask_rows(bool valid, const BB<G::W>& legal,
                                                      bool pass_bit) {
    constexpr int NW = (G::A + 31) / 32, STRIDE = NW + 1;
    __shared__ u32 stage[(LX_BLOCK / 32) * 32 * STRIDE];
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    u32* mine = stage + (warp * 32 + lane) * STRIDE;
    if (G::IDENT) {
#pragma unroll
        for (int j = 0; j < NW; j++) {
            u32 v = j < G::W ? legal.w[j] : 0u;
            if (G::PASS >= 0 && j == (G::C >> 5) && pass_bit) v |= 1u << (G::C & 31);
            mine[j] = valid ? v : 0u;
        }
    } else {                                   // embedded layout: compact bits to cell order
        for (int j = 0; j < NW; j++) mine[j] = 0u;
        if (valid) {
            for (int c = 0; c < G::C; c++)
                if (test(legal, G::cell_bit(c))) mine[c >> 5] |= 1u << (c & 31);
            if (G::PASS >= 0 && pass_bit) mine[G::C >> 5] |= 1u << (G::C & 31);
        }
    }
    mine[NW] = 0u;
    __syncwarp();
    return stage + warp * 32 * STRIDE;
}

// Warp-cooperative write of the (B, A) uint8 legal mask for the warp's 32
// consecutive envs: the rows staged as bit vectors (stage_mask_rows) form
// one contiguous block of 32*A bytes in global memory, written with
// coalesced 16-byte stores.  Every lane of the warp must call it (rows >= B
// pass valid = false).
template <class G>
__device__ __forceinline__ void write_mask_rows(unsigned char* __restrict__ mask, i64 B, i64 i,
                                                bool valid, const BB<G::W>& legal,
                                                bool pass_bit) {
    constexpr int A = G::A, NW = (G::A + 31) / 32, STRIDE = NW + 1;
    const u32* rows = stage_mask_rows<G>(valid, legal, pass_bit);
    const unsigned lane = threadIdx.x & 31u;
    const i64 i0 = i - lane;
    const i64 left = B - i0;
    const int nrows = left < 32 ? (int)left : 32;
    const int bytes = nrows * A;
    unsigned char* base = mask + i0 * (i64)A;
#if LX_MASK_STREAM
    // (A <= 128: the stream block stays small beside the big boards' row
    // mirror in the 48 KB of static shared memory)
    if (A <= 128 && nrows == 32) {
        // full warp: concatenate the 32 rows into one bit stream (row r at bit
        // r*A; each lane ORs its row's words in at their offset), so the 2A
        // 16-byte output pieces are 16-aligned halves of stream words -- no
        // row-crossing walk per piece (r2z ncu: that walk was ~40 % of the C4
        // env step's instructions)
        constexpr int SW = A <= 128 ? A + 1 : 1;
        __shared__ u32 stream_all[(LX_BLOCK / 32) * SW];
        u32* S = stream_all + (threadIdx.x >> 5) * SW;
        for (int k = (int)lane; k < SW; k += 32) S[k] = 0u;
        __syncwarp();
        const u32* mine = rows + lane * STRIDE;
        const int q0 = (int)lane * A;
#pragma unroll
        for (int j = 0; j < NW; j++) {
            const u32 v = mine[j];
            if (v) {
                const int q = q0 + 32 * j;
                const int w = q >> 5, sh = q & 31;
                atomicOr(&S[w], v << sh);
                if (sh) atomicOr(&S[w + 1], v >> (32 - sh));
            }
        }
        __syncwarp();
        for (int k = (int)lane; k < 2 * A; k += 32) {
            const u32 v = (S[k >> 1] >> ((k & 1) << 4)) & 0xffffu;
            *reinterpret_cast<uint4*>(base + 16 * k) =
                make_uint4(spread4(v), spread4(v >> 4), spread4(v >> 8), spread4(v >> 12));
        }
        __syncwarp();
        return;
    }
#endif
    for (int p0 = (int)lane * 16; p0 < bytes; p0 += 32 * 16) {
        const int nb = bytes - p0 < 16 ? bytes - p0 : 16;
        u32 v = 0u;
        int got = 0, r = p0 / A, c = p0 - r * A;
        while (got < nb) {
            const int take = (nb - got) < (A - c) ? (nb - got) : (A - c);
            const u32* rw = rows + r * STRIDE;
            const u32 lo = rw[c >> 5], hi = rw[(c >> 5) + 1];
            const u32 bits = __funnelshift_r(lo, hi, (unsigned)(c & 31)) & ((1u << take) - 1u);
            v |= bits << got;
            got += take;
            r++;
            c = 0;
        }
        if (nb == 16) {
            *reinterpret_cast<uint4*>(base + p0) =
                make_uint4(spread4(v), spread4(v >> 4), spread4(v >> 8), spread4(v >> 12));
        } else {
            for (int j = 0; j < nb; j++) base[p0 + j] = (v >> j) & 1u;
        }
    }
    __syncwarp();
}

// Bit-packed legal mask: (B, NW) u32 rows, action a = bit a%32 of word a/32
// (NW = ceil(A/32)).  The warp's 32 rows are one contiguous block of 32*NW
// words, copied from the staged rows with coalesced 4-byte stores.
template <class G>
__device__ __forceinline__ void write_mask_bits(u32* __restrict__ mask, i64 B, i64 i, bool valid,
                                                const BB<G::W>& legal, bool pass_bit) {
    constexpr int NW = (G::A + 31) / 32, STRIDE = NW + 1;
    if constexpr (G::IDENT && (NW == 1 || NW == 2 || NW == 4) && NW >= G::W) {
        // rows of 4 / 8 / 16 bytes: each lane stores its own row with one
        // vector store (consecutive lanes, consecutive rows: coalesced)
        if (valid) {
            u32 v[NW];
#pragma unroll
            for (int j = 0; j < NW; j++) {
                v[j] = j < G::W ? legal.w[j] : 0u;
                if (G::PASS >= 0 && j == (G::C >> 5) && pass_bit) v[j] |= 1u << (G::C & 31);
            }
            if constexpr (NW == 1) mask[i] = v[0];
            else if constexpr (NW == 2) reinterpret_cast<uint2*>(mask)[i] = make_uint2(v[0], v[1]);
            else reinterpret_cast<uint4*>(mask)[i] = make_uint4(v[0], v[1], v[2], v[3]);
        }
        return;
    }
    const u32* rows = stage_mask_rows<G>(valid, legal, pass_bit);
    const unsigned lane = threadIdx.x & 31u;
    const i64 i0 = i - lane;
    const i64 left = B - i0;
    const int nrows = left < 32 ? (int)left : 32;
    u32* base = mask + i0 * (i64)NW;
    for (int k = (int)lane; k < nrows * NW; k += 32) base[k] = rows[(k / NW) * STRIDE + k % NW];
    __syncwarp();
}

// Movement / gridworld masks (A = C*C or #directions): the warp zeroes its 32
// contiguous rows with 16-byte stores, then each lane sets the bytes of its
// own legal actions (a few dozen per row).  Every lane of the warp must call.
template <class G>
__device__ __forceinline__ void write_mask_moves(unsigned char* __restrict__ mask, i64 B, i64 i,
                                                 bool valid, const typename G::St& s, bool live,
                                                 bool pass_bit) {
    constexpr int A = G::A;
    const unsigned lane = threadIdx.x & 31u;
    const i64 i0 = i - lane;
    const i64 left = B - i0;
    const int nrows = left < 32 ? (int)left : 32;
    const i64 bytes = (i64)nrows * A;
    unsigned char* base = mask + i0 * (i64)A;
    const i64 n16 = bytes >> 4;
    uint4* b16 = reinterpret_cast<uint4*>(base);
    for (i64 q = lane; q < n16; q += 32) b16[q] = make_uint4(0u, 0u, 0u, 0u);
    for (i64 p = (n16 << 4) + lane; p < bytes; p += 32) base[p] = 0;
    __syncwarp();
    if (valid) {
        unsigned char* row = mask + i * (i64)A;
        if (live) G::enum_moves(s, [&](int a) { row[a] = 1; });
        if (G::PASS >= 0 && pass_bit) row[G::PASS] = 1;
    }
    __syncwarp();
}

// Bit-packed movement / gridworld masks: the warp zeroes its 32 contiguous
// rows of NW words, then each lane sets the bits of its own legal actions.
template <class G>
__device__ __forceinline__ void write_mask_moves_bits(u32* __restrict__ mask, i64 B, i64 i,
                                                      bool valid, const typename G::St& s,
                                                      bool live, bool pass_bit) {
    constexpr int NW = (G::A + 31) / 32;
    const unsigned lane = threadIdx.x & 31u;
    const i64 i0 = i - lane;
    const i64 left = B - i0;
    const int nrows = left < 32 ? (int)left : 32;
    u32* base = mask + i0 * (i64)NW;
    for (int k = (int)lane; k < nrows * NW; k += 32) base[k] = 0u;
    __syncwarp();
    if (valid) {
        u32* row = mask + i * (i64)NW;
        if (live) G::enum_moves(s, [&](int a) { row[a >> 5] |= 1u << (a & 31); });
        if (G::PASS >= 0 && pass_bit) row[G::PASS >> 5] |= 1u << (G::PASS & 31);
    }
    __syncwarp();
}

// Coalesced (B, N)-byte row output for 128-thread blocks (lx_export,
// lx_observe): each lane fills its row in a per-warp shared-memory stage
// (pitch NP bytes = an odd number of words, so the 32 lanes' byte stores hit
// 32 different banks), then the warp writes the 32 rows -- consecutive lanes
// on consecutive bytes -- to dst + row * stride, so every store instruction
// covers whole sectors instead of 32 rows C bytes apart.  All lanes call.
template <int PITCH>
struct RowStage {
    static constexpr int NP = (((PITCH + 3) / 4) | 1) * 4;
    static constexpr int BYTES = 4 * 32 * NP;
    static __device__ __forceinline__ unsigned char* row() {
        __shared__ __align__(16) unsigned char buf[BYTES];
        return buf + ((threadIdx.x >> 5) & 3) * 32 * NP + (threadIdx.x & 31u) * NP;
    }
    // the first N (<= PITCH) bytes of the warp's rows [i0, i0 + 32) to dst
    // (row pitch `stride` bytes)
    template <int N>
    static __device__ __forceinline__ void flush(unsigned char* __restrict__ dst, i64 stride,
                                                 i64 B, i64 i) {
        __syncwarp();
        const unsigned lane = threadIdx.x & 31u;
        const i64 i0 = i - lane;
        const i64 left = B - i0;
        const int nrows = left < 32 ? (int)left : 32;
        const unsigned char* base = row() - lane * NP;
        if (stride == N && ((reinterpret_cast<unsigned long long>(dst + i0 * (i64)N) & 3ull) == 0)) {
            // rows back to back: the warp's block is contiguous; when it starts
            // on a 4-byte boundary (the caller's array usually does, and i0 is
            // a multiple of 32) it goes out as 4-byte stores
            u32* d4 = reinterpret_cast<u32*>(dst + i0 * (i64)N);
            const int nbytes = nrows * N, nw = nbytes >> 2;
            for (int q = (int)lane; q < nw; q += 32) {
                u32 v = 0u;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const int p = 4 * q + k, r = p / N, c = p - r * N;
                    v |= (u32)base[r * NP + c] << (8 * k);
                }
                d4[q] = v;
            }
            for (int p = 4 * nw + (int)lane; p < nbytes; p += 32) {
                const int r = p / N, c = p - r * N;
                dst[i0 * (i64)N + p] = base[r * NP + c];
            }
        } else {
            for (int q = (int)lane; q < nrows * N; q += 32) {
                const int r = q / N, c = q - r * N;
                dst[(i0 + r) * stride + c] = base[r * NP + c];
            }
        }
        __syncwarp();
    }
};

}  // namespace lx


// ---------------------------------------------------------------- kernels
//
// The native runtime compiles the kernels in groups, one NVRTC program per
// group in parallel (LX_GROUP = group id; unset: every kernel):
//   0 init / rollout / export / import   1 legal / sample / observe
//   2 verify / step / random_step        3 expand (MCTS)   4 env_step   5 mcts
#ifndef LX_GROUP
#define LX_GROUP -1
#endif
#define LX_IN_GROUP(g) (LX_GROUP < 0 || LX_GROUP == (g))

// Envs per thread of the per-ply kernels (lx_random_step, lx_env_step):
// each thread loads K envs before working on any of them (block b covers
// envs [b*256*K, (b+1)*256*K), slot j of thread t is env b*256*K + j*256 +
// t).  K = 2 was measured slower on the B200 (r2d: C4 env step 52.8 -> 47.4 G
// env steps/s with bit masks): with 32-48 B states these kernels are issue-
// and register-bound (ncu: issue 55-65 %, math-pipe throttle the top stall,
// occupancy limited by registers), not short of bytes in flight.
// minimum resident blocks per SM of the per-ply HBM kernels: a register
// cap that buys occupancy (r2k A/B at 4: Hex env step +11 %, Reversi +12 %,
// C4 / TTT / Pente even; 6 spills)
#ifndef LX_STEP_MINB
#define LX_STEP_MINB 4
#endif
#ifndef LX_STEP_K_OVERRIDE
#define LX_STEP_K_OVERRIDE 1
#endif
#ifndef LX_STEP_K
#define LX_STEP_K (LX_STEP_K_OVERRIDE)
#endif

struct LxRefPtrs {               // reference GameState field pointers (state.py:78-130)
    signed char* board_piece;    // (B, C) int8, -1 empty
    signed char* board_owner;    // (B, C) int8, -1 empty
    signed char* current_player; // (B,)
    int* move_count;             // (B,) int32
    unsigned char* terminated;   // (B,) bool
    unsigned char* truncated;    // (B,) bool
    signed char* outcome;        // (B,) int8
    unsigned long long* seeds;   // (B,) uint64
    int* scores;                 // (B, 2) int32        or null
    short* pass_streak;          // (B,) int16          or null
    unsigned char* pass_flags;   // (B, 2) bool         or null
    signed char* last_mover;     // (B,) int8           or null
    signed char* last_kind;      // (B,) int8
    short* last_source;          // (B,) int16
    short* last_dest;            // (B,) int16
    short* last_dest_by_player;  // (B, 2) int16
    short* comp_labels;          // (B, P, C) int16     or null (P connectivity plans)
    signed char* phase;          // (B,) int8           or null
    short* must_move;            // (B,) int16          or null
    signed char* turn_pos;       // (B,) int8           or null
    unsigned char* hopped_mask;  // (B, C) bool         or null (transient masks)
    unsigned char* captured_mask;
    unsigned char* promoted_mask;
};

#if LX_IN_GROUP(0)
extern "C" __global__ void __launch_bounds__(LX_BLOCK) lx_init(u32* st, i64 B, const u64* seeds,
                                                          u64 seed_base, i64 first) {
    const i64 i = lx::gtid();
    if (i >= B) return;
    Game::St s;
    const u64 seed = seeds ? seeds[i] : lx::mix64(lx::seed_mix(seed_base) ^ (u64)(first + i));
    lx::init_state<Game>(s, seed);
    lx::store_state<Game>(s, st, B, i);
}
#endif

// Static facts of the game and of its device state layout, read by the
// native runtime at lx_game_create (lx_game_info, include/ludax_b200.h).
#if LX_IN_GROUP(0)
extern "C" __constant__ int lx_facts[10] = {
    Game::C, Game::A, Game::PASS, Game::W, lx::Layout<Game>::NQ, Game::NX, Game::MECH,
    lx::Layout<Game>::NWORDS, LX_STEP_K, LX_BLOCK};

// mark rows (uint8 (B,), null = all) that are still live terminated +
// truncated with a draw outcome (engine.playout_random's cap, engine.py:156-160;
// the MCTS stuck / cap handling, agents.py:430-435)
extern "C" __global__ void __launch_bounds__(LX_BLOCK) lx_truncate(u32* st, i64 B,
                                                              const unsigned char* rows) {
    const i64 i = lx::gtid();
    if (i >= B || (rows && !rows[i])) return;
    Game::St s;
    lx::load_state<Game>(s, st, B, i);
    if (s.term) return;
    s.term = 1; s.trunc = 1; s.outcome = 0;
    lx::store_state<Game>(s, st, B, i);
}

// replace every row's RNG seed (the MCTS rollout re-keying, agents.py:229-233)
extern "C" __global__ void __launch_bounds__(LX_BLOCK) lx_set_seeds(u32* st, i64 B, const u64* seeds) {
    const i64 i = lx::gtid();
    if (i >= B) return;
    Game::St s;
    lx::load_state<Game>(s, st, B, i);
    s.seed = seeds[i];
    lx::store_state<Game>(s, st, B, i);
}
#endif

// (B, A) uint8 mask (null to skip) and (B,) int64 counts (null to skip);
// terminated rows are all-false / zero (reference compiler.py:394-428).
// mover (B,) int8 or null: legality for that player instead of the row's
// current player, in the row's phase (the reference's `mover=` argument).
#if LX_IN_GROUP(1)
extern "C" __global__ void __launch_bounds__(LX_BLOCK) lx_legal(const u32* st, i64 B,
                                                           const signed char* mover,
                                                           unsigned char* mask, i64* counts) {
    const i64 i = lx::gtid();
    if ((i64)(blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) >= B) return;   // whole warp out
    const bool valid = i < B;
    bool pass_only = false;
    if constexpr (Game::MECH == 0) {
        lx::BB<Game::W> legal = lx::bb_zero<Game::W>();
        if (valid) {
            Game::St s;
            lx::load_state<Game>(s, st, B, i);
            if (mover) s.cur = mover[i];
            if (!s.term) legal = Game::legal(s);
            const int n = lx::popc(legal);
            pass_only = !s.term && n == 0 && Game::force_pass(s.phase);
            if (counts) counts[i] = s.term ? 0 : (pass_only ? 1 : n);
        }
        if (mask) lx::write_mask_rows<Game>(mask, B, i, valid, legal, pass_only);
    } else {
        Game::St s;
        bool live = false;
        if (valid) {
            lx::load_state<Game>(s, st, B, i);
            if (mover) s.cur = mover[i];
            live = !s.term;
            const int n = live ? lx::legal_count<Game>(s) : 0;
            pass_only = live && n == 0 && Game::force_pass(s.phase);
            if (counts) counts[i] = !live ? 0 : (pass_only ? 1 : n);
        }
        if (mask) lx::write_mask_moves<Game>(mask, B, i, valid, s, live, pass_only);
    }
}
#endif

// sampled action per row from u (when given) or from the row's own stream;
// mover as in lx_legal
#if LX_IN_GROUP(1)
extern "C" __global__ void __launch_bounds__(LX_BLOCK) lx_sample(const u32* st, i64 B,
                                                            const signed char* mover,
                                                            const double* u, i64* actions) {
    const i64 i = lx::gtid();
    if (i >= B) return;
    Game::St s;
    lx::load_state<Game>(s, st, B, i);
    if (mover) s.cur = mover[i];
    if (s.term) { actions[i] = -1; return; }
    if (!u) { actions[i] = lx::sample_action<Game>(s, lx::seed_mix(s.seed)); return; }
    if constexpr (Game::MECH == 0) {
        const lx::BB<Game::W> legal = Game::legal(s);
        const int n = lx::popc(legal);
        if (n == 0) { actions[i] = Game::force_pass(s.phase) ? Game::PASS : -1; return; }
        i64 r = __double2ll_rz(__dmul_rn(u[i], (double)n));
        r = r < (i64)(n - 1) ? r : (i64)(n - 1);
        actions[i] = Game::bit_cell(lx::select_bit(legal, (int)r));
    } else {
        int tot[Game::NG];
        const int n = Game::count_moves(s, tot);
        if (n == 0) { actions[i] = Game::force_pass(s.phase) ? Game::PASS : -1; return; }
        i64 r = __double2ll_rz(__dmul_rn(u[i], (double)n));
        r = r < (i64)(n - 1) ? r : (i64)(n - 1);
        int hint;
        actions[i] = Game::select_move(s, (int)r, tot, hint);
    }
}
#endif

// verification pass: *bad = min illegal live row (init to ~0 by the caller)
#if LX_IN_GROUP(2)
extern "C" __global__ void __launch_bounds__(LX_BLOCK) lx_verify(const u32* st, i64 B,
                                                            const i64* actions,
                                                            const unsigned char* rows,
                                                            u64* bad) {
    const i64 i = lx::gtid();
    if (i >= B) return;
    if (rows && !rows[i]) return;
    Game::St s;
    lx::load_state<Game>(s, st, B, i);
    if (s.term) return;
    if (!lx::action_legal<Game>(s, actions[i])) atomicMin(bad, (u64)i);
}
#endif

// in-place step of live rows (rows & ~terminated)
#if LX_IN_GROUP(2)
extern "C" __global__ void __launch_bounds__(LX_BLOCK) lx_step(u32* st, i64 B, const i64* actions,
                                                          const unsigned char* rows) {
    const i64 i = lx::gtid();
    if (i >= B) return;
    if (rows && !rows[i]) return;
    Game::St s;
    lx::load_state<Game>(s, st, B, i);
    if (s.term) return;
    lx::apply_step<Game>(s, (int)actions[i]);
    lx::store_state<Game>(s, st, B, i);
}
#endif

// fused sample+step for live rows, one ply (engine.random_actions + step_into)
#if LX_IN_GROUP(2)
extern "C" __global__ void __launch_bounds__(LX_BLOCK, LX_STEP_MINB) lx_random_step(u32* st, i64 B, int max_turns,
                                                                 i64* actions_out) {
    constexpr int K = LX_STEP_K;
    const i64 base = (i64)blockIdx.x * blockDim.x * K + threadIdx.x;
    Game::St s[K];
#pragma unroll
    for (int j = 0; j < K; j++) {
        const i64 i = base + (i64)j * blockDim.x;
        if (i < B) lx::load_state<Game>(s[j], st, B, i);
    }
#pragma unroll
    for (int j = 0; j < K; j++) {
        const i64 i = base + (i64)j * blockDim.x;
        if (i >= B) continue;
        if (s[j].term || (int)s[j].mc >= max_turns) {
            if (actions_out) actions_out[i] = -1;
            continue;
        }
        int hint;
        const int a = lx::sample_action<Game>(s[j], lx::seed_mix(s[j].seed), hint);
        if (actions_out) actions_out[i] = a;
        if (a < 0) continue;
        lx::apply_step<Game>(s[j], a, hint);
        lx::store_state<Game>(s[j], st, B, i);
    }
}
#endif

// Fused rollout.  Persistent threads: each thread plays one env at a time to
// the end with the whole state in registers, then starts another, so no lane
// idles while a long game finishes.
//   mode & 1: start each env from its seed (seeds[i] or spawn(seed_base, first+i))
//             else load it from st
//   mode & 2: store the final state to st
//   mode & 4: truncate unfinished envs at max_turns (engine.playout_random)
// stats (u64[8], written by the last block): steps, p1 wins, p2 wins, draws,
// truncated, envs finished, lowest row that had no legal action (~0: none).
//
// Game-over handling is batched per warp: a lane whose game ends keeps its
// final state in registers and waits until LX_REFILL_LANES lanes are waiting
// (or LX_REFILL_WAIT plies passed, or nothing else is running); then every
// waiting lane flushes (stats, final-state store) and starts its next env in
// one pass, instead of one or two lanes running that code every ply.
#ifndef LX_ROLLOUT_THREADS
#define LX_ROLLOUT_THREADS 256
#endif
#ifndef LX_ROLLOUT_MINB
#define LX_ROLLOUT_MINB 2
#endif
#ifndef LX_REFILL_LANES
#define LX_REFILL_LANES 6
#endif
#ifndef LX_REFILL_WAIT
#define LX_REFILL_WAIT 6
#endif
#ifndef LX_PLY_UNROLL
#define LX_PLY_UNROLL 1
#endif
// small grids (grid x threads >= B, i.e. every env fits one wave of the
// persistent threads): warp w plays env chunk w with no claim atomics, and a
// one-block launch publishes its stats without the cross-block ticket
#ifndef LX_STATIC_CHUNKS
#define LX_STATIC_CHUNKS 1
#endif
// grids of 2..8 blocks launched as one cluster publish through distributed
// shared memory (the host sets the cluster dimension; without it the ticket
// path below runs)
#ifndef LX_CLUSTER_PUBLISH
#define LX_CLUSTER_PUBLISH 1
#endif
// cross-block publish ordered by one acq_rel ticket atomic instead of two
// sequentially consistent fences (__threadfence)
#ifndef LX_ACQREL_TICKET
#define LX_ACQREL_TICKET 1
#endif
#if LX_IN_GROUP(0)
namespace lx {
// End of a rollout launch: warp sums -> stats (u64[8]) and a cleared work
// buffer.  Out of line by default so that the epilogue's code does not
// perturb the register allocation of the ply loop (inlined, the cluster path
// cost C4 three registers: 64 -> 67, one block per SM fewer); the row-mirror
// games inline it (Pente: 124 registers out of line, 103 inlined = one more
// 128-thread block per SM).  The lowering picks LX_PUBLISH_INLINE per game.
#ifndef LX_PUBLISH_INLINE
#define LX_PUBLISH_INLINE 0
#endif
#if LX_PUBLISH_INLINE
#define LX_PUBLISH_ATTR __forceinline__
#else
#define LX_PUBLISH_ATTR __noinline__
#endif
__device__ LX_PUBLISH_ATTR void publish_stats(u32 n_steps, u32 n_p1, u32 n_p2, u32 n_draw,
                                           u32 n_trunc, u32 n_done, u64* stats, u64* work) {
    u64* counter = work;
    u64* stuck_max = work + 1;
    u64* acc = work + 2;
    const unsigned lane = threadIdx.x & 31u;
    // warp reduce, one atomic per warp per counter
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_steps += __shfl_xor_sync(0xffffffffu, n_steps, o);
        n_p1 += __shfl_xor_sync(0xffffffffu, n_p1, o);
        n_p2 += __shfl_xor_sync(0xffffffffu, n_p2, o);
        n_draw += __shfl_xor_sync(0xffffffffu, n_draw, o);
        n_trunc += __shfl_xor_sync(0xffffffffu, n_trunc, o);
        n_done += __shfl_xor_sync(0xffffffffu, n_done, o);
    }
    // a grid that is one block, or one thread-block cluster (the host
    // launches grids of 2..8 blocks as a single cluster): per-block sums in
    // shared memory, rank 0 adds the cluster's blocks through distributed
    // shared memory -- no ticket, no fences, no global atomics
    // (a block plays <= blockDim.x envs of <= max_turns plies: u32 sums)
    u32 ncta = 1;
    if (LX_CLUSTER_PUBLISH && gridDim.x > 1 && gridDim.x <= 8)
        asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
    if ((LX_STATIC_CHUNKS && gridDim.x == 1) || (ncta > 1 && ncta == gridDim.x)) {
        __shared__ u32 blk[6];
        if (threadIdx.x < 6) blk[threadIdx.x] = 0u;
        __syncthreads();
        if (lane == 0) {
            atomicAdd(&blk[0], n_steps);
            atomicAdd(&blk[1], n_p1);
            atomicAdd(&blk[2], n_p2);
            atomicAdd(&blk[3], n_draw);
            atomicAdd(&blk[4], n_trunc);
            atomicAdd(&blk[5], n_done);
        }
        if (ncta > 1) {
            // release/acquire at cluster scope: every block's sums and stuck /
            // stall atomics are visible to rank 0 after the barrier
            asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                         "barrier.cluster.wait.acquire.aligned;" ::: "memory");
            if (blockIdx.x == 0 && threadIdx.x < 6) {
                const u32 local = (u32)__cvta_generic_to_shared(&blk[threadIdx.x]);
                u64 sum = 0;
                for (u32 r = 0; r < ncta; r++) {
                    u32 remote, v;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                                 : "=r"(remote) : "r"(local), "r"(r));
                    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote));
                    sum += v;
                }
                stats[threadIdx.x] = sum;
            }
        } else {
            __syncthreads();
            if (threadIdx.x < 6) stats[threadIdx.x] = (u64)blk[threadIdx.x];
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            const u64 sm = atomicExch(stuck_max, 0ull);
            stats[6] = sm ? ~sm : ~0ull;
            stats[7] = atomicExch(work + 9, 0ull);       // seed-upload stall (0: none)
            *counter = 0ull;
        }
        if (ncta > 1)                  // keep every block's shared memory until rank 0 read it
            asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                         "barrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    if (lane == 0) {
        atomicAdd(acc + 0, (u64)n_steps);
        atomicAdd(acc + 1, (u64)n_p1);
        atomicAdd(acc + 2, (u64)n_p2);
        atomicAdd(acc + 3, (u64)n_draw);
        atomicAdd(acc + 4, (u64)n_trunc);
        atomicAdd(acc + 5, (u64)n_done);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#if LX_ACQREL_TICKET
        // release: this block's sums (ordered before it by the barrier,
        // cumulatively) precede the ticket; acquire: the last block sees
        // every block's sums
        u64 ticket;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;"
                     : "=l"(ticket) : "l"(work + 8) : "memory");
#else
        __threadfence();
        const u64 ticket = atomicAdd(work + 8, 1ull);
#endif
        if (ticket == (u64)gridDim.x - 1) {            // last block: publish, then clear
#if !LX_ACQREL_TICKET
            __threadfence();
#endif
#pragma unroll
            for (int k = 0; k < 6; k++) stats[k] = atomicExch(acc + k, 0ull);
            const u64 sm = atomicExch(stuck_max, 0ull);
            stats[6] = sm ? ~sm : ~0ull;               // lowest stuck row, ~0 = none
            stats[7] = atomicExch(work + 9, 0ull);       // seed-upload stall (0: none)
            atomicExch(counter, 0ull);
            atomicExch(work + 8, 0ull);
        }
    }
}

template <bool STREAM>
__device__ __forceinline__ void rollout_body(u32* st, i64 B, int max_turns, int mode,
                                             u64 seed_base, const u64* seeds, i64 first,
                                             u64* stats, u64* work, signed char* outcomes,
                                             int* turns, const u32* ready) {
    // work (u64[16], zero on entry, left zero on exit): [0] env-chunk counter,
    // [1] ~(lowest stuck row) by atomicMax (0 = none), [2..7] stats being
    // accumulated, [8] finished-block ticket, [9] seed-upload stall flag.  The
    // last block to finish moves the sums to `stats` and clears `work`, so a
    // launch needs no memsets.
    // STREAM (lx_rollout_streamed): the seeds are still being uploaded
    // (lx_playout_host): *ready counts the 32-env chunks already in HBM (the
    // copy stream writes it after each piece), so a warp waits for its chunk
    // before reading the seeds -- the upload overlaps the play instead of
    // preceding it.
    u64* counter = work;
    u64* stuck_max = work + 1;
    u64* acc = work + 2;
    constexpr unsigned FULL = 0xffffffffu;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned lanes_below = (1u << lane) - 1u;
    const u64 base_mix = lx::seed_mix(seed_base);
    u32 n_steps = 0, n_p1 = 0, n_p2 = 0, n_draw = 0, n_trunc = 0, n_done = 0;
    // Env indices are handed out in warp-private chunks of 32, the next chunk
    // claimed once the current one is half used (its atomic's latency hides
    // behind ~16 games); each lane precomputes the seed (and its first mix)
    // of env chunk+lane at full warp width and a lane starting a game fetches
    // its seed with a shuffle.
    auto prep = [&](u64 base, u64& ps, u64& pm) {
        const i64 j = (i64)(base + lane);
        ps = 0;
        pm = 0;
        if (STREAM && (mode & 1) && base < (u64)B) {                 // warp-uniform
            const u64 last = base + 31 < (u64)B ? base + 31 : (u64)B - 1;
            const u32 need = (u32)(last >> 5) + 1u;
            if (lane == 0) {
                // bounded: after 4 s the launch gives up waiting (sticky flag,
                // reported in stats[7]) instead of hanging on a stalled copy
                const u64 t0 = lx::globaltimer_ns();
                volatile const u64* stalled = work + 9;
                while (lx::ld_acquire_gpu(ready) < need && *stalled == 0ull) {
                    __nanosleep(128);
                    if (lx::globaltimer_ns() - t0 > 4000000000ull) {
                        atomicOr(work + 9, 1ull);
                        break;
                    }
                }
            }
            __syncwarp();
        }
        if ((mode & 1) && j < B) {
            // streamed seeds are read from L2 (the DMA wrote them after launch)
            ps = seeds ? (STREAM ? __ldcg(seeds + j) : seeds[j])
                       : lx::mix64(base_mix ^ (u64)(first + j));
            pm = lx::seed_mix(ps);
        }
    };
    u64 cur = 0, nxt = 0;
    bool requested = false;       // next chunk claimed (warp-uniform)
    // grid-uniform: the whole batch is one wave of warps (host sizes the grid
    // as min(resident blocks, ceil(B / threads)))
    const bool static_chunks = LX_STATIC_CHUNKS &&
                               (u64)gridDim.x * blockDim.x >= (u64)B;
    if (static_chunks) {
        cur = (u64)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
        nxt = (u64)B;             // "next chunk" is past the end: nothing to claim
        requested = true;
    } else {
        if (lane == 0) cur = atomicAdd(counter, 32ull);
        cur = __shfl_sync(FULL, cur, 0);
    }
    int used = 0;
    u64 pre_seed, pre_mix;
    prep(cur, pre_seed, pre_mix);
    Game::St s;
    u64 smix = 0;
    i64 idx = -1;
    // lane flags as 32-bit ints: bools live in byte lanes of a register and
    // every update costs a PRMT on the ALU pipe
    int playing = 0, pending = 0, active = 1;
    int waited = 0;               // plies since a lane started waiting (warp-uniform)
    while (true) {
        const unsigned idle = __ballot_sync(FULL, active && !playing);
        const unsigned busy = __ballot_sync(FULL, playing);
        if (idle && (__popc(idle) >= LX_REFILL_LANES || waited >= LX_REFILL_WAIT || !busy)) {
            waited = 0;
            const bool me = (idle >> lane) & 1u;
            if (me && pending) {                        // flush the finished game
                if ((mode & 4) && !s.term) { s.term = 1; s.trunc = 1; s.outcome = 0; }
                n_p1 += s.outcome == 1;
                n_p2 += s.outcome == 2;
                n_draw += s.outcome == 0;
                n_trunc += s.trunc;
                n_done += 1;
                if (mode & 2) lx::store_state<Game>(s, st, B, idx);
                if (outcomes) outcomes[idx] = (signed char)s.outcome;
                if (turns) turns[idx] = (int)s.mc;
                pending = false;
            }
            const int n = __popc(idle);
            const int pos = used + __popc(idle & lanes_below);
            u64 sd = __shfl_sync(FULL, pre_seed, pos & 31);
            u64 sm = __shfl_sync(FULL, pre_mix, pos & 31);
            u64 my_base = cur;
            if (used + n > 32) {                        // switch to the next chunk
                // (a warp past the end claims nothing more: static chunks
                // never touch the counter)
                if (!requested && lane == 0) nxt = cur < (u64)B ? atomicAdd(counter, 32ull) : (u64)B;
                requested = false;
                const u64 nb = __shfl_sync(FULL, nxt, 0);
                u64 ps2, pm2;
                prep(nb, ps2, pm2);
                const u64 sd2 = __shfl_sync(FULL, ps2, pos & 31);
                const u64 sm2 = __shfl_sync(FULL, pm2, pos & 31);
                if (pos >= 32) { sd = sd2; sm = sm2; my_base = nb; }
                cur = nb;
                used = used + n - 32;
                pre_seed = ps2;
                pre_mix = pm2;
            } else {
                used += n;
            }
            if (!requested && used >= 16 && cur < (u64)B) {
                if (lane == 0) nxt = atomicAdd(counter, 32ull);
                requested = true;
            }
            if (me) {
                idx = (i64)(my_base + (u64)(pos & 31));
                if (idx >= B) {
                    active = false;
                } else {
                    if (mode & 1) {
                        lx::init_state<Game>(s, sd);
                        smix = sm;
                    } else {
                        lx::load_state<Game>(s, st, B, idx);
                        smix = lx::seed_mix(s.seed);
                    }
                    playing = !(s.term || (int)s.mc >= max_turns);
                    pending = !playing;
                }
            }
        } else if (idle) {
            waited++;
        }
        if (!__any_sync(FULL, active)) break;
        // LX_PLY_UNROLL plies per pass of the refill bookkeeping above (its
        // ballots and branches are warp-wide overhead paid once per pass; a
        // lane whose game ends on an earlier ply idles for the rest of it)
#pragma unroll
        for (int u = 0; u < LX_PLY_UNROLL; u++) {
            if constexpr (Game::SPLIT_FLOOD) {
                // reach-set games: the ply is split around its flood, which the
                // whole warp runs converged (lx::coop_flood) -- inside a ply
                // only the playing lanes are active and each would flood alone
                typename Game::Flood fl;
                fl.need = 0;
                fl.f = lx::bb_zero<Game::W>();
                fl.free_ = fl.f;
                int a = -1;
                if (playing) {
                    int hint;
                    a = lx::sample_action<Game>(s, smix, hint);
                    if (a >= 0) lx::apply_step_pre<Game>(s, a, fl);
                }
                lx::coop_flood<Game::W>(fl.need != 0, fl.free_, fl.f,
                                        [](const lx::LW<Game::W>& x) { return Game::flood_dil(x); });
                if (playing) {
                    if (a < 0) {
                        atomicMax(stuck_max, ~(u64)idx);
                        playing = 0;
                        pending = 1;
                    } else {
                        lx::apply_step_post<Game>(s, a, fl);
                        n_steps++;
                        if (s.term || (int)s.mc >= max_turns) {
                            playing = 0;
                            pending = 1;
                        }
                    }
                }
            } else {
                if (playing) {
                    int hint;
                    const int a = lx::sample_action<Game>(s, smix, hint);
                    if (a < 0) {
                        atomicMax(stuck_max, ~(u64)idx);
                        playing = 0;
                        pending = 1;
                    } else {
                        lx::apply_step<Game>(s, a, hint);
                        n_steps++;
                        if (s.term || (int)s.mc >= max_turns) {
                            playing = 0;
                            pending = 1;
                        }
                    }
                }
            }
        }
    }
    publish_stats(n_steps, n_p1, n_p2, n_draw, n_trunc, n_done, stats, work);
}

}  // namespace lx

extern "C" __global__ void __launch_bounds__(LX_ROLLOUT_THREADS, LX_ROLLOUT_MINB)
lx_rollout(u32* st, i64 B, int max_turns, int mode, u64 seed_base, const u64* seeds, i64 first,
           u64* stats, u64* work, signed char* outcomes, int* turns) {
    lx::rollout_body<false>(st, B, max_turns, mode, seed_base, seeds, first, stats, work,
                            outcomes, turns, nullptr);
}

// the same rollout while lx_playout_host streams the seeds up (see STREAM)
extern "C" __global__ void __launch_bounds__(LX_ROLLOUT_THREADS, LX_ROLLOUT_MINB)
lx_rollout_streamed(u32* st, i64 B, int max_turns, int mode, u64 seed_base, const u64* seeds,
                    i64 first, u64* stats, u64* work, signed char* outcomes, int* turns,
                    const u32* ready) {
    lx::rollout_body<true>(st, B, max_turns, mode, seed_base, seeds, first, stats, work,
                           outcomes, turns, ready);
}

#endif

// MCTS expansion + rollout, one thread per expanded child (reference
// agents._Search._attach_and_rollout + _rollout, agents.py:211-238, 313-353).
// States live in a node pool (quad-major, row stride `cap`): child row
// children[i] = parent row parents[i] stepped with actions[i].  Per child:
// info[i] = current_player | terminated << 2 | (outcome + 1) << 3 |
// legal count << 8, its (A,) legal mask row in masks (when non-null), and
// when it is live and has a legal action, the outcome of one uniform-random
// rollout from it drawing with seeds[i] (0 draw / stuck / cap, 1 P1, 2 P2)
// in rolled[i] (else -1).
#if LX_IN_GROUP(5)
namespace lx {

// ---- device MCTS (one thread per search tree) --------------------------------
// The reference's UCB1 search (agents._Search, agents.py:84-310) per tree:
// forced prefix of root expansions, then iterations of selection / one-child
// expansion / uniform-random rollout / backpropagation, then the best root
// child.  Trees are independent, so one thread running its tree's iterations
// in order reproduces the reference's lockstep batches exactly.  Node states
// live in a pool (row = tree * nmax + node); node records and action lists
// in a per-tree arena.  UCB arithmetic is IEEE double with no contraction
// (--fmad=false) and log(N) from a host table, so every comparison matches
// the reference's Python floats.
struct MctsNode {
    int N, to_move, term, outcome, stuck, nacts, nexp, acts;   // acts: arena offset (-1: unbuilt)
    double W;
};

template <class G>
__device__ __forceinline__ int mcts_legal(const typename G::St& s, int* out) {
    int n = 0;
    if (s.term) return 0;
    if constexpr (G::MECH == 0) {
        const BB<G::W> legal = G::legal(s);
#pragma unroll
        for (int w = 0; w < G::W; w++) {
            u32 b = legal.w[w];
            while (b) { const int x = 32 * w + __ffs(b) - 1; b &= b - 1u; out[n++] = G::bit_cell(x); }
        }
    } else {
        G::enum_moves(s, [&](int a) { out[n++] = a; });
    }
    if (n == 0 && G::PASS >= 0 && G::force_pass(s.phase)) out[n++] = G::PASS;
    return n;
}

// one uniform-random rollout from s drawing with `seed` (agents._rollout):
// 0 draw / cap / stuck, 1 P1, 2 P2.  Out of line: the MCTS kernel calls it
// from two places and inlining the rules twice doubles its compile time.
template <class G>
__device__ __noinline__ int mcts_playout(typename G::St& s, u64 seed, int max_turns) {
    s.seed = seed;
    s.ncached = 0;
    const u64 smix = seed_mix(seed);
    while (!s.term && (int)s.mc < max_turns) {
        int hint;
        const int a = sample_action<G>(s, smix, hint);
        if (a < 0) break;                          // stuck: scored as a draw
        apply_step<G>(s, a, hint);
    }
    return s.term && !s.trunc ? s.outcome : 0;
}

}  // namespace lx

// One warp per search tree (block t = tree t).  The tree -- node records,
// action lists, child lists and, when `smem` is set, the node states -- lives
// in dynamic shared memory (else in the per-tree global arena / node pool).
// Every lane runs the search on the same data (so control flow is uniform
// and the per-lane registers agree); lane 0 alone writes the tree, followed
// by __syncwarp, and the lanes split the work that is parallel: the UCB1
// scores of a node's children (reduced to the best by (score desc, action
// asc), the reference's order) and the rank sort of a new node's actions.
// status[t]: 0 ok, 1 arena or path capacity exceeded (the caller falls back)
extern "C" __global__ void __launch_bounds__(32) lx_mcts(
        const u32* roots, i64 n, const u64* keys, const int* budgets, double c,
        int rollout_max_turns, const double* logs, int nlogs, u32* pool, i64 pool_rows, int nmax,
        unsigned char* arena, i64 arena_bytes, i64* actions_out, int* status, int smem) {
    const i64 t = blockIdx.x;
    if (t >= n) return;
    const int lane = (int)(threadIdx.x & 31u);
    const bool L0 = lane == 0;
    constexpr unsigned FULL = 0xffffffffu;
    using lx::MctsNode;
    typedef Game::St St;
    constexpr int MAXPATH = 256;
    constexpr int NQW = lx::Layout<Game>::NQ * 4;
    extern __shared__ __align__(16) unsigned char lx_mcts_smem[];
    unsigned char* ar = smem ? lx_mcts_smem : arena + t * arena_bytes;
    MctsNode* nodes = reinterpret_cast<MctsNode*>(ar);
    int* acts = reinterpret_cast<int*>(nodes + nmax);
    // ints: acts + kids, then (A + 1) u64 sort keys and (A + 1) ints of sort output
    const i64 sort_bytes = (i64)(Game::A + 1) * 12;
    const i64 acap = (arena_bytes - (i64)nmax * (i64)sizeof(MctsNode) - sort_bytes) / 8;
    int* kids = acts + acap;
    u64* hk = reinterpret_cast<u64*>(kids + acap);
    int* sorted = reinterpret_cast<int*>(hk + (Game::A + 1));
    u32* sstates = reinterpret_cast<u32*>(ar + arena_bytes);   // smem: node states after the arena
    i64 aused = 0;
    if (L0) status[t] = 0;
    const u64 key = keys[t];
    const int budget = budgets[t];
    const u64 k0 = lx::mix64(lx::HASH_SEED ^ key);
    const u64 k_order = lx::mix64(k0 ^ 0xA11ull), k_roll = lx::mix64(k0 ^ 0x5011ull),
              k_best = lx::mix64(k0 ^ 0x7Eull);
    const i64 base = t * (i64)nmax;
    int nnodes = 0;
    bool overflow = false;

    auto load_node = [&](int node, St& s) {
        if (smem) {
            u32 w[NQW];
#pragma unroll
            for (int k = 0; k < NQW; k++) w[k] = sstates[(i64)node * NQW + k];
            lx::unpack<Game>(s, w);
        } else {
            lx::load_state<Game>(s, pool, pool_rows, base + node);
        }
    };
    auto store_node = [&](int node, const St& s) {     // lane 0 (caller syncs)
        if (smem) {
            u32 w[NQW];
            lx::pack<Game>(s, w);
#pragma unroll
            for (int k = 0; k < NQW; k++) sstates[(i64)node * NQW + k] = w[k];
        } else {
            lx::store_state<Game>(s, pool, pool_rows, base + node);
        }
    };
    auto meta = [&](MctsNode& nd, const St& s) {       // lane 0 (caller syncs)
        nd.N = 0; nd.W = 0.0; nd.to_move = s.cur; nd.term = s.term; nd.outcome = s.outcome;
        nd.nacts = 0; nd.nexp = 0; nd.acts = -1;
    };
    // untried order: legal actions sorted by hash_key(key, 0xA11, a), ties by
    // a, duplicates dropped: lane 0 lists the actions, the lanes hash and rank
    // a stripe each, lane 0 compacts
    auto build = [&](int node, const St& s) {
        MctsNode& nd = nodes[node];
        int* out = acts + aused;
        if (aused + Game::A + 1 > acap) {
            overflow = true;
            if (L0) { nd.acts = (int)aused; nd.nacts = 0; }
            __syncwarp();
            return;
        }
        int m = 0;
        if (L0) m = lx::mcts_legal<Game>(s, out);
        m = __shfl_sync(FULL, m, 0);
        __syncwarp();
        for (int i = lane; i < m; i += 32) hk[i] = lx::mix64(k_order ^ (u64)(i64)out[i]);
        __syncwarp();
        for (int i = lane; i < m; i += 32) {
            const u64 h = hk[i];
            const int a = out[i];
            int rank = 0;
            for (int j = 0; j < m; j++) {
                const u64 hj = hk[j];
                const int aj = out[j];
                rank += (hj < h || (hj == h && (aj < a || (aj == a && j < i))));
            }
            sorted[rank] = a;
        }
        __syncwarp();
        int u = 0;
        if (L0) {
            for (int i = 0; i < m; i++)
                if (u == 0 || out[u - 1] != sorted[i]) out[u++] = sorted[i];
            nd.acts = (int)aused;
            nd.nacts = u;
        }
        u = __shfl_sync(FULL, u, 0);
        __syncwarp();
        aused += u;
    };
    auto value_for = [](int player, int outcome) -> double {
        if (outcome == 0) return 0.0;
        return outcome == player + 1 ? 1.0 : -1.0;
    };
    int path[MAXPATH];
    auto backprop = [&](int len, int outcome) {
        if (L0) {
            nodes[path[0]].N += 1;
            for (int i = 1; i < len; i++) {
                nodes[path[i]].N += 1;
                nodes[path[i]].W += value_for(nodes[path[i - 1]].to_move, outcome);
            }
        }
        __syncwarp();
    };
    // child of `parent` by its next untried action; returns the backed-up value
    auto expand = [&](int parent, int action, int& child, u64 rkey, bool do_roll) -> int {
        St s;
        load_node(parent, s);
        if (!s.term) lx::apply_step<Game>(s, action);
        child = nnodes++;
        int cnt = 0;
        if (!s.term) {
            cnt = lx::legal_count<Game>(s);
            if (cnt == 0 && Game::PASS >= 0 && Game::force_pass(s.phase)) cnt = 1;
        }
        if (L0) {
            store_node(child, s);
            MctsNode& nd = nodes[child];
            meta(nd, s);
            nd.stuck = !s.term && cnt == 0;
            kids[nodes[parent].acts + nodes[parent].nexp] = child;
            nodes[parent].nexp += 1;
        }
        __syncwarp();
        if (s.term || cnt == 0 || !do_roll) return s.outcome;
        return lx::mcts_playout<Game>(s, rkey, rollout_max_turns);
    };

    {   // root
        St s;
        lx::load_state<Game>(s, roots, n, t);
        if (L0) { store_node(0, s); meta(nodes[0], s); }
        __syncwarp();
        nnodes = 1;
        build(0, s);
        if (L0) nodes[0].stuck = nodes[0].nacts == 0;
        __syncwarp();
    }
    const MctsNode& root = nodes[0];
    int nodes_created = 0;
    // forced prefix: the first min(budget, branching) root children, rollouts
    // keyed by the node count after the whole batch is attached
    int start_it = 0;
    if (!root.term && !root.stuck) {
        const int k = budget < root.nacts ? budget : root.nacts;
        const u64 rk = lx::mix64(k_roll ^ (u64)k);
        int first = nnodes;
        for (int j = 0; j < k; j++) {
            int child;
            expand(0, acts[root.acts + j], child, rk, false);
        }
        nodes_created = k;
        for (int j = 0; j < k; j++) {             // rollouts + backprop in attach order
            const int child = first + j;
            const MctsNode& nd = nodes[child];
            int outcome = nd.outcome;
            if (!nd.term && !nd.stuck) {
                St s;
                load_node(child, s);
                outcome = lx::mcts_playout<Game>(s, rk, rollout_max_turns);
            }
            path[0] = 0; path[1] = child;
            backprop(2, outcome);
        }
        start_it = k;
    }
    for (int it = start_it; it < budget && !overflow; it++) {
        int node = 0, len = 1;
        path[0] = 0;
        while (true) {
            const MctsNode& nd = nodes[node];
            if (nd.term || nd.stuck) { backprop(len, nd.term ? nd.outcome : 0); break; }
            if (nd.acts < 0) {
                St s;
                load_node(node, s);
                build(node, s);
                if (overflow) break;
                if (nd.nacts == 0 && nd.nexp == 0) {
                    if (L0) nodes[node].stuck = 1;
                    __syncwarp();
                    continue;
                }
            }
            if (nd.nexp < nd.nacts) {
                if (nnodes >= nmax || len + 1 >= MAXPATH) { overflow = true; break; }
                nodes_created += 1;
                int child;
                const int outcome = expand(node, acts[nd.acts + nd.nexp], child,
                                           lx::mix64(k_roll ^ (u64)nodes_created), true);
                path[len++] = child;
                backprop(len, outcome);
                break;
            }
            // UCB1 over the expanded children, lanes over a stripe each, then
            // the warp's best by (score desc, action asc)
            const double log_n = logs[nd.N < nlogs ? nd.N : nlogs - 1];
            int best = -1, best_a = 0x7fffffff;
            double best_s = 0.0;
            for (int j = lane; j < nd.nexp; j += 32) {
                const int kid = kids[nd.acts + j];
                const MctsNode& ch = nodes[kid];
                const double sc = ch.W / (double)ch.N + c * sqrt(log_n / (double)ch.N);
                const int a = acts[nd.acts + j];
                if (best < 0 || sc > best_s || (sc == best_s && a < best_a)) {
                    best = kid; best_s = sc; best_a = a;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double os = __shfl_xor_sync(FULL, best_s, o);
                const int oa = __shfl_xor_sync(FULL, best_a, o);
                const int ob = __shfl_xor_sync(FULL, best, o);
                if (ob >= 0 && (best < 0 || os > best_s || (os == best_s && oa < best_a))) {
                    best = ob; best_s = os; best_a = oa;
                }
            }
            if (len >= MAXPATH) { overflow = true; break; }
            node = best;
            path[len++] = node;
        }
    }
    if (overflow) {
        if (L0) { status[t] = 1; actions_out[t] = -1; }
        return;
    }
    // best root child: (N, mean value, seeded draw), insertion order, strict >
    i64 best_a = -1;
    if (root.nexp == 0) {
        best_a = root.nacts > 0 ? acts[root.acts] : -1;
    } else {
        int bN = -1;
        double bQ = 0.0, bU = 0.0;
        for (int j = 0; j < root.nexp; j++) {
            const MctsNode& ch = nodes[kids[root.acts + j]];
            const int a = acts[root.acts + j];
            const double q = ch.W / (double)(ch.N > 1 ? ch.N : 1);
            const double u = lx::key_uniform(lx::mix64(k_best ^ (u64)(i64)a));
            const bool better = bN < 0 || ch.N > bN || (ch.N == bN && (q > bQ || (q == bQ && u > bU)));
            if (better) { bN = ch.N; bQ = q; bU = u; best_a = a; }
        }
    }
    if (L0) actions_out[t] = best_a;
}
#endif

#if LX_IN_GROUP(3)
extern "C" __global__ void __launch_bounds__(128) lx_expand(u32* pool, i64 cap, const i64* parents,
                                                            const i64* actions,
                                                            const i64* children, i64 n,
                                                            const u64* seeds, int max_turns,
                                                            int* info, signed char* rolled,
                                                            unsigned char* masks) {
    const i64 i = lx::gtid();
    if (i >= n) return;
    Game::St s;
    lx::load_state<Game>(s, pool, cap, parents[i]);
    if (!s.term) lx::apply_step<Game>(s, (int)actions[i]);
    lx::store_state<Game>(s, pool, cap, children[i]);
    int cnt = 0;
    bool pass_only = false;
    if (!s.term) {
        cnt = lx::legal_count<Game>(s);
        pass_only = cnt == 0 && Game::force_pass(s.phase);
        if (pass_only) cnt = 1;
    }
    info[i] = s.cur | (s.term << 2) | ((s.outcome + 1) << 3) | (cnt << 8);
    if (masks) {
        unsigned char* row = masks + i * (i64)Game::A;
        for (int a = 0; a < Game::A; a++) row[a] = 0;
        if (!s.term) {
            if constexpr (Game::MECH == 0) {
                const lx::BB<Game::W> legal = Game::legal(s);
                for (int c = 0; c < Game::C; c++) row[c] = lx::test(legal, Game::cell_bit(c));
            } else {
                Game::enum_moves(s, [&](int a) { row[a] = 1; });
            }
            if (Game::PASS >= 0 && pass_only) row[Game::PASS] = 1;
        }
    }
    signed char out = -1;
    if (!s.term && cnt > 0) {
        s.seed = seeds[i];
        s.ncached = 0;
        const u64 smix = lx::seed_mix(s.seed);
        while (!s.term && (int)s.mc < max_turns) {
            int hint;
            const int a = lx::sample_action<Game>(s, smix, hint);
            if (a < 0) break;                      // stuck: scored as a draw
            lx::apply_step<Game>(s, a, hint);
        }
        out = (signed char)(s.term && !s.trunc ? s.outcome : 0);
    }
    rolled[i] = out;
}
#endif

// PGX-style environment step (env.LudaxEnvironment.step), one launch per ply.
// flags: LX_ENV_STEP apply one ply to live rows (else only refresh outputs);
// LX_ENV_RANDOM sample a uniform legal action in the kernel from the row's
// own stream (engine.random_actions; written to `actions` when non-null)
// instead of reading `actions`; LX_ENV_AUTO_RESET re-initialise finished
// rows with seed hash_key(seed, 0xE9) (engine.reset_rows, engine.py:58-65);
// LX_ENV_MASK_BITS write the mask as (B, ceil(A/32)) u32 bit rows instead of
// (B, A) uint8.  Rewards of the terminating ply follow the outcome (reference
// engine.py:79-87: P1 win [+1,-1], P2 win [-1,+1], draw [0,0]); games that
// reach max_turns (> 0) are truncated draws.  With auto-reset the
// terminating ply's terminated / truncated / rewards are reported while the
// stored state, mask and player are the reset env's (PGX auto_reset).  An
// illegal given action (reference engine.step raises IllegalAction,
// mechanics.py:503-510) is not applied: the row ends with the PGX
// illegal-action penalty (mover -1, opponent +1, outcome = opponent win) and
// *bad receives the lowest such row; a random row with no legal action and
// no pass (EmptyMask, engine.py:142-147) ends as a truncated draw and is
// reported the same way.
#define LX_ENV_AUTO_RESET 1
#define LX_ENV_RANDOM 2
#define LX_ENV_MASK_BITS 4
#define LX_ENV_STEP 8
#if LX_IN_GROUP(4)
namespace lx {
// one env of lx_env_step: apply / sample, rewards, flags, auto-reset; leaves
// the next state's legality for the mask writer in legal / pass_only / live
template <class G>
__device__ __forceinline__ void env_step_one(typename G::St& s, u32* st, i64 B, i64 i,
                                             i64* actions, int max_turns, int flags,
                                             float* rewards, unsigned char* terminated,
                                             unsigned char* truncated, int* player, u64* bad,
                                             bool want_mask, BB<G::W>& legal, bool& pass_only,
                                             bool& live) {
    float r0 = 0.f, r1 = 0.f;
    bool out_term = s.term, out_trunc = s.trunc;
    if ((flags & LX_ENV_STEP) && !s.term) {
        int a, hint = -1;
        bool ok;
        if (flags & LX_ENV_RANDOM) {
            a = sample_action<G>(s, seed_mix(s.seed), hint);
            if (actions) actions[i] = a;
            ok = a >= 0;
        } else {
            const i64 a64 = actions[i];
            ok = action_legal<G>(s, a64);
            a = (int)a64;
        }
        if (ok) {
            apply_step<G>(s, a, hint);
            if (s.term) {
                r0 = s.outcome == 1 ? 1.f : (s.outcome == 2 ? -1.f : 0.f);
                r1 = -r0;
            } else if (max_turns > 0 && (int)s.mc >= max_turns) {
                s.term = 1; s.trunc = 1; s.outcome = 0;
            }
        } else {
            if (bad) atomicMin(bad, (u64)i);
            s.term = 1;
            if (flags & LX_ENV_RANDOM) {               // stuck: truncated draw
                s.trunc = 1; s.outcome = 0;
            } else {                                   // illegal: the mover loses
                s.outcome = 2 - s.cur;
                r0 = s.cur ? 1.f : -1.f;
                r1 = -r0;
            }
        }
        out_term = s.term;
        out_trunc = s.trunc;
        if ((flags & LX_ENV_AUTO_RESET) && s.term) {
            const u64 seed = mix64(seed_mix(s.seed) ^ 0xE9ull);
            init_state<G>(s, seed);
        }
        store_state<G>(s, st, B, i);
    }
    if (rewards) reinterpret_cast<float2*>(rewards)[i] = make_float2(r0, r1);
    if (terminated) terminated[i] = (unsigned char)out_term;
    if (truncated) truncated[i] = (unsigned char)out_trunc;
    if (player) player[i] = s.cur;
    live = !s.term;
    if constexpr (G::MECH == 0) {
        if (want_mask && live) legal = G::legal(s);
        pass_only = live && !any(legal) && G::force_pass(s.phase);
    } else {
        if (want_mask && live) pass_only = legal_count<G>(s) == 0 && G::force_pass(s.phase);
    }
}
}  // namespace lx

extern "C" __global__ void __launch_bounds__(LX_BLOCK, LX_STEP_MINB) lx_env_step(u32* st, i64 B, i64* actions,
                                                              int max_turns, int flags,
                                                              void* mask, float* rewards,
                                                              unsigned char* terminated,
                                                              unsigned char* truncated,
                                                              int* player, u64* bad) {
    constexpr int K = LX_STEP_K;
    const i64 base = (i64)blockIdx.x * blockDim.x * K + threadIdx.x;
    Game::St s[K];
#pragma unroll
    for (int j = 0; j < K; j++) {
        const i64 i = base + (i64)j * blockDim.x;
        if (i < B) lx::load_state<Game>(s[j], st, B, i);
    }
#pragma unroll
    for (int j = 0; j < K; j++) {
        const i64 i = base + (i64)j * blockDim.x;
        if (i - (i64)(threadIdx.x & 31u) >= B) continue;        // whole warp out (uniform)
        const bool valid = i < B;
        lx::BB<Game::W> legal = lx::bb_zero<Game::W>();
        bool pass_only = false, live = false;
        if (valid)
            lx::env_step_one<Game>(s[j], st, B, i, actions, max_turns, flags, rewards,
                                   terminated, truncated, player, bad, mask != nullptr, legal,
                                   pass_only, live);
        if (mask) {
            if (flags & LX_ENV_MASK_BITS) {
                if constexpr (Game::MECH == 0)
                    lx::write_mask_bits<Game>((u32*)mask, B, i, valid, legal, pass_only);
                else
                    lx::write_mask_moves_bits<Game>((u32*)mask, B, i, valid, s[j], live,
                                                    pass_only);
            } else {
                if constexpr (Game::MECH == 0)
                    lx::write_mask_rows<Game>((unsigned char*)mask, B, i, valid, legal,
                                              pass_only);
                else
                    lx::write_mask_moves<Game>((unsigned char*)mask, B, i, valid, s[j], live,
                                               pass_only);
            }
        }
    }
}
#endif

// device state -> reference GameState SoA (state.py:78-130)
#if LX_IN_GROUP(0)
extern "C" __global__ void __launch_bounds__(128) lx_export(const u32* st, i64 B, LxRefPtrs p) {
    const i64 i = lx::gtid();
    if ((i64)(blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) >= B) return;   // whole warp out
    const bool valid = i < B;
    Game::St s;
    if (valid) lx::load_state<Game>(s, st, B, i);
    // one stage, wide enough for int16 label rows when they fit in 48 KB
    constexpr bool STAGE_LABELS = Game::L_CONN && lx::RowStage<2 * Game::C>::BYTES <= 48 * 1024;
    typedef lx::RowStage<STAGE_LABELS ? 2 * Game::C : Game::C> Rows;
    unsigned char* r = Rows::row();
    if (p.board_owner) {                       // null: scalar fields only (B200Game.meta)
        if (valid)
            for (int c = 0; c < Game::C; c++) {
                const int cb = Game::cell_bit(c);
                r[c] = lx::test(s.own0, cb) ? 0 : (lx::test(s.own1, cb) ? 1 : 0xff);
            }
        Rows::template flush<Game::C>((unsigned char*)p.board_owner, Game::C, B, i);
        if (valid)
            for (int c = 0; c < Game::C; c++) {
                const int cb = Game::cell_bit(c);
                r[c] = (lx::test(s.own0, cb) || lx::test(s.own1, cb))
                           ? (unsigned char)Game::piece_at(s, cb) : 0xff;
            }
        Rows::template flush<Game::C>((unsigned char*)p.board_piece, Game::C, B, i);
    }
    if (p.hopped_mask) {
        unsigned char* outs[3] = {p.hopped_mask, p.captured_mask, p.promoted_mask};
        for (int k = 0; k < 3; k++) {
            if (valid) {
                unsigned char h[Game::C], cm[Game::C], pm[Game::C];
                Game::export_transient(s, h, cm, pm);
                const unsigned char* src = k == 0 ? h : (k == 1 ? cm : pm);
                for (int c = 0; c < Game::C; c++) r[c] = src[c];
            }
            Rows::template flush<Game::C>(outs[k], Game::C, B, i);
        }
    }
    if constexpr (Game::L_CONN) {
        if (p.comp_labels) {                   // (B, P, C) int16 rows
            if constexpr (STAGE_LABELS) {      // staged plan by plan
                short lab[Game::CONN_PLANS * Game::C];
                if (valid) Game::labels(s, lab);
                for (int k = 0; k < Game::CONN_PLANS; k++) {
                    short* rs = reinterpret_cast<short*>(r);
                    if (valid)
                        for (int c = 0; c < Game::C; c++) rs[c] = lab[k * Game::C + c];
                    Rows::template flush<2 * Game::C>((unsigned char*)p.comp_labels + 2 * k * Game::C,
                                                      2 * Game::CONN_PLANS * Game::C, B, i);
                }
            } else if (valid) {
                Game::labels(s, p.comp_labels + i * Game::CONN_PLANS * Game::C);
            }
        }
    }
    if (!valid) return;
    if (p.current_player) p.current_player[i] = (signed char)s.cur;
    if (p.move_count) p.move_count[i] = (int)s.mc;
    if (p.terminated) p.terminated[i] = (unsigned char)s.term;
    if (p.truncated) p.truncated[i] = (unsigned char)s.trunc;
    if (p.outcome) p.outcome[i] = (signed char)s.outcome;
    if (p.seeds) p.seeds[i] = s.seed;
    if (p.scores) { p.scores[2 * i] = s.sc0; p.scores[2 * i + 1] = s.sc1; }
    if (p.pass_streak) {
        p.pass_streak[i] = (short)s.pass_streak;
        p.pass_flags[2 * i] = (unsigned char)s.pf0;
        p.pass_flags[2 * i + 1] = (unsigned char)s.pf1;
    }
    if (p.last_mover) {
        p.last_mover[i] = (signed char)s.last_mover;
        p.last_kind[i] = (signed char)s.last_kind;
        p.last_source[i] = (short)s.last_source;
        p.last_dest[i] = (short)s.last_dest;
        p.last_dest_by_player[2 * i] = (short)s.ldbp0;
        p.last_dest_by_player[2 * i + 1] = (short)s.ldbp1;
    }
    if (p.phase) p.phase[i] = (signed char)s.phase;
    if (p.must_move) p.must_move[i] = (short)s.must_move;
    if (p.turn_pos) p.turn_pos[i] = (signed char)s.pos;
}
#endif

// reference GameState SoA -> device state (inverse of lx_export)
#if LX_IN_GROUP(0)
extern "C" __global__ void __launch_bounds__(128) lx_import(u32* st, i64 B, LxRefPtrs p) {
    const i64 i = lx::gtid();
    if (i >= B) return;
    Game::St s;
    lx::init_state<Game>(s, p.seeds[i]);
    s.own0 = lx::bb_zero<Game::W>();
    s.own1 = lx::bb_zero<Game::W>();
    const signed char* own = p.board_owner + i * Game::C;
    const signed char* pc = p.board_piece + i * Game::C;
    Game::clear_types(s);
    for (int c = 0; c < Game::C; c++) {
        if (own[c] == 0) lx::setbit(s.own0, Game::cell_bit(c));
        else if (own[c] == 1) lx::setbit(s.own1, Game::cell_bit(c));
        if (own[c] >= 0) Game::set_piece(s, Game::cell_bit(c), pc[c]);
    }
    s.cur = p.current_player[i];
    s.mc = (u32)p.move_count[i];
    s.term = p.terminated[i];
    s.trunc = p.truncated[i];
    s.outcome = p.outcome[i];
    s.sc0 = p.scores ? p.scores[2 * i] : 0;
    s.sc1 = p.scores ? p.scores[2 * i + 1] : 0;
    if (p.pass_streak) {
        s.pass_streak = p.pass_streak[i];
        s.pf0 = p.pass_flags[2 * i];
        s.pf1 = p.pass_flags[2 * i + 1];
    }
    if (p.last_mover) {
        s.last_mover = p.last_mover[i];
        s.last_kind = p.last_kind[i];
        s.last_source = p.last_source[i];
        s.last_dest = p.last_dest[i];
        s.ldbp0 = p.last_dest_by_player[2 * i];
        s.ldbp1 = p.last_dest_by_player[2 * i + 1];
    }
    s.phase = p.phase ? p.phase[i] : 0;
    s.must_move = p.must_move ? p.must_move[i] : -1;
    s.pos = p.turn_pos ? p.turn_pos[i] : 0;
    if (p.hopped_mask) Game::import_transient(s, p.hopped_mask + i * Game::C,
                                              p.captured_mask + i * Game::C,
                                              p.promoted_mask + i * Game::C);
    Game::rebuild_ext(s);
    lx::store_state<Game>(s, st, B, i);
}
#endif

// (B, 2T+1, C) uint8 relative-owner planes (reference compiler.py:611-626):
// per piece type t the player's and the opponent's pieces of type t, then
// the is-mover plane
#if LX_IN_GROUP(1)
extern "C" __global__ void __launch_bounds__(128) lx_observe(const u32* st, i64 B, int player,
                                                             unsigned char* planes) {
    const i64 i = lx::gtid();
    if ((i64)(blockIdx.x * blockDim.x + (threadIdx.x & ~31u)) >= B) return;   // whole warp out
    const bool valid = i < B;
    Game::St s;
    if (valid) lx::load_state<Game>(s, st, B, i);
    constexpr int T = Game::NT;
    constexpr i64 ROW = (i64)(2 * T + 1) * Game::C;
    typedef lx::RowStage<Game::C> Rows;
    unsigned char* r = Rows::row();
    for (int k = 0; k < 2 * T + 1; k++) {      // plane by plane, each staged then flushed
        if (valid) {
            if (k == 2 * T) {
                const unsigned char mv = s.cur == player;
                for (int c = 0; c < Game::C; c++) r[c] = mv;
            } else {
                const lx::BB<Game::W> tb = Game::type_bb(s, k >> 1);
                const lx::BB<Game::W> side = ((k & 1) ^ player) ? s.own1 : s.own0;
                const lx::BB<Game::W> b = side & tb;
                for (int c = 0; c < Game::C; c++) r[c] = lx::test(b, Game::cell_bit(c));
            }
        }
        Rows::template flush<Game::C>(planes + k * Game::C, ROW, B, i);
    }
}
#endif
