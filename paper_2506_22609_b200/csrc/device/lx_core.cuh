// lx_core.cuh -- bitboard, RNG and sampling primitives for the per-game
// NVRTC translation units (sm_100a).  Self-contained: no CUDA or libc
// headers, so NVRTC compiles it without an include path to the toolkit.
//
// Board encoding: one bit per cell in row-major cell order (cell i is bit
// i%32 of 32-bit word i/32).  Bit order == cell order, which is what makes
// "r-th set bit" equal the reference's "r-th legal cell in ascending index"
// (reference mechanics.py:488-492).
#pragma once

typedef unsigned int u32;
typedef unsigned long long u64;
typedef long long i64;

namespace lx {

template <int W>
struct BB {
    u32 w[W];
};

template <int W>
__device__ __forceinline__ BB<W> bb_zero() {
    BB<W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = 0u;
    return r;
}

template <int W>
__device__ __forceinline__ BB<W> operator&(const BB<W>& a, const BB<W>& b) {
    BB<W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = a.w[i] & b.w[i];
    return r;
}
template <int W>
__device__ __forceinline__ BB<W> operator|(const BB<W>& a, const BB<W>& b) {
    BB<W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = a.w[i] | b.w[i];
    return r;
}
template <int W>
__device__ __forceinline__ BB<W> operator^(const BB<W>& a, const BB<W>& b) {
    BB<W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = a.w[i] ^ b.w[i];
    return r;
}
// a & ~b
template <int W>
__device__ __forceinline__ BB<W> andnot(const BB<W>& a, const BB<W>& b) {
    BB<W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = a.w[i] & ~b.w[i];
    return r;
}
template <int W>
__device__ __forceinline__ bool any(const BB<W>& a) {
    u32 o = 0u;
#pragma unroll
    for (int i = 0; i < W; i++) o |= a.w[i];
    return o != 0u;
}
template <int W>
__device__ __forceinline__ bool equal(const BB<W>& a, const BB<W>& b) {
    u32 o = 0u;
#pragma unroll
    for (int i = 0; i < W; i++) o |= a.w[i] ^ b.w[i];
    return o == 0u;
}
template <int W>
__device__ __forceinline__ int popc(const BB<W>& a) {
    int n = 0;
#pragma unroll
    for (int i = 0; i < W; i++) n += __popc(a.w[i]);
    return n;
}
// select without dynamic register indexing: s ? b : a
template <int W>
__device__ __forceinline__ BB<W> sel(bool s, const BB<W>& a, const BB<W>& b) {
    BB<W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = s ? b.w[i] : a.w[i];
    return r;
}

// Powers of two as run-time constants (constant bank): a funnel shift by a
// constant written as multiplies by these stays on the FMA pipe as IMAD /
// IMAD.HI with a constant-bank operand -- the compiler cannot strength-reduce
// a multiplier it does not know back into an ALU shift.
#ifndef LX_SHIFT_FMA
#define LX_SHIFT_FMA 0
#endif
#if LX_SHIFT_FMA && defined(__CUDA_ARCH__)
__constant__ u32 lx_pow2[32] = {
    1u << 0, 1u << 1, 1u << 2, 1u << 3, 1u << 4, 1u << 5, 1u << 6, 1u << 7,
    1u << 8, 1u << 9, 1u << 10, 1u << 11, 1u << 12, 1u << 13, 1u << 14, 1u << 15,
    1u << 16, 1u << 17, 1u << 18, 1u << 19, 1u << 20, 1u << 21, 1u << 22, 1u << 23,
    1u << 24, 1u << 25, 1u << 26, 1u << 27, 1u << 28, 1u << 29, 1u << 30, 1u << 31};
// (hi:lo) >> s, low word, for 0 < s < 32: umulhi(lo, 2^(32-s)) + hi * 2^(32-s)
// (the two parts occupy disjoint bits, so + is |)
__device__ __forceinline__ u32 fshr_fma(u32 lo, u32 hi, unsigned s) {
    const u32 m = lx_pow2[32 - s];
    return __umulhi(lo, m) + hi * m;
}
// (hi:lo) << s, high word: hi * 2^s + umulhi(lo, 2^s)
__device__ __forceinline__ u32 fshl_fma(u32 lo, u32 hi, unsigned s) {
    const u32 m = lx_pow2[s];
    return hi * m + __umulhi(lo, m);
}
#define LX_FSHR(lo, hi, s) fshr_fma((lo), (hi), (s))
#define LX_FSHL(lo, hi, s) fshl_fma((lo), (hi), (s))
#else
#define LX_FSHR(lo, hi, s) __funnelshift_r((lo), (hi), (s))
#define LX_FSHL(lo, hi, s) __funnelshift_l((lo), (hi), (s))
#endif

// gather: result bit x = a bit (x + S).  S > 0 moves bits towards lower
// indices.  Caller masks with the direction's validity mask.
template <int W, int S>
__device__ __forceinline__ BB<W> gather(const BB<W>& a) {
    BB<W> r;
    if constexpr (S == 0) {
        return a;
    } else if constexpr (S > 0) {
        constexpr int q = S / 32;
        constexpr unsigned s = (unsigned)(S % 32);
#pragma unroll
        for (int i = 0; i < W; i++) {
            const u32 lo = (i + q < W) ? a.w[i + q] : 0u;
            const u32 hi = (i + q + 1 < W) ? a.w[i + q + 1] : 0u;
            r.w[i] = s ? LX_FSHR(lo, hi, s) : lo;
        }
    } else {
        constexpr int q = (-S) / 32;
        constexpr unsigned s = (unsigned)((-S) % 32);
#pragma unroll
        for (int i = 0; i < W; i++) {
            const u32 hi = (i - q >= 0) ? a.w[i - q] : 0u;
            const u32 lo = (i - q - 1 >= 0) ? a.w[i - q - 1] : 0u;
            r.w[i] = s ? LX_FSHL(lo, hi, s) : hi;
        }
    }
    return r;
}

// dynamic single-bit helpers (cell index c known only at run time); written
// as unrolled compare/select so the board never leaves registers
template <int W>
__device__ __forceinline__ BB<W> onehot(int c) {
    BB<W> r;
    const u32 word = (u32)c >> 5, bit = 1u << (c & 31);
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = (word == (u32)i) ? bit : 0u;
    return r;
}
template <int W>
__device__ __forceinline__ bool test(const BB<W>& a, int c) {
    const u32 word = (u32)c >> 5;
    u32 v = 0u;
#pragma unroll
    for (int i = 0; i < W; i++) v = (word == (u32)i) ? a.w[i] : v;
    return (v >> (c & 31)) & 1u;
}
template <int W>
__device__ __forceinline__ void setbit(BB<W>& a, int c) {
    const u32 word = (u32)c >> 5, bit = 1u << (c & 31);
#pragma unroll
    for (int i = 0; i < W; i++) a.w[i] |= (word == (u32)i) ? bit : 0u;
}
// set bit c in b when side (0/1) is 1, else in a.  The side mask is built
// arithmetically (0 - side) rather than from a predicate, so each board word
// is one LOP3 (a | (v & ~m), b | (v & m)) instead of a select per word and
// board (C4: 8 SEL + 4 LOP -> 4 LOP3 per ply).
template <int W>
__device__ __forceinline__ void place_bit(BB<W>& a, BB<W>& b, int c, int side) {
    const u32 word = (u32)c >> 5, bit = 1u << (c & 31);
#if defined(__CUDA_ARCH__)
    u32 m;
    asm("sub.u32 %0, 0, %1;" : "=r"(m) : "r"((u32)side));   // opaque: no predicate rewrite
#else
    const u32 m = 0u - (u32)side;
#endif
#pragma unroll
    for (int i = 0; i < W; i++) {
        const u32 v = (word == (u32)i) ? bit : 0u;
        a.w[i] |= v & ~m;
        b.w[i] |= v & m;
    }
}
template <int W>
__device__ __forceinline__ void clearbit(BB<W>& a, int c) {
    const u32 word = (u32)c >> 5, bit = 1u << (c & 31);
#pragma unroll
    for (int i = 0; i < W; i++) a.w[i] &= (word == (u32)i) ? ~bit : 0xffffffffu;
}

// nibble j of Sel8::v[b] = position of the j-th set bit of byte b
struct Sel8 {
    u32 v[256];
    __host__ __device__ constexpr Sel8() : v() {
        for (int b = 0; b < 256; b++) {
            u32 t = 0u;
            int j = 0;
            for (int p = 0; p < 8; p++)
                if ((b >> p) & 1) { t |= (u32)p << (4 * j); j++; }
            v[b] = t;
        }
    }
};
__device__ const Sel8 lx_sel8 = Sel8();

#ifndef LX_SELECT_SWAR
#define LX_SELECT_SWAR 1
#endif
#ifndef LX_SELECT_STASH
#define LX_SELECT_STASH 1
#endif
#if LX_SELECT_SWAR
// position of the r-th (0-based) set bit of a 32-bit word; r < popc(x).
// SWAR byte popcounts, their inclusive prefix sums by one multiply, the byte
// holding the bit from a byte-parallel compare, then a 256-entry table for
// the bit inside that byte (~20 instructions, a third of them off the ALU
// pipe, vs ~35 ALU for the 5-level binary search below)
__device__ __forceinline__ int select32(u32 x, int r) {
    u32 b = x - ((x >> 1) & 0x55555555u);
    b = (b & 0x33333333u) + ((b >> 2) & 0x33333333u);
    b = (b + (b >> 4)) & 0x0f0f0f0fu;
    const u32 pre = b * 0x01010101u;                    // byte k: popc of bytes 0..k
    const u32 ge = ((pre | 0x80808080u) - (u32)(r + 1) * 0x01010101u) & 0x80808080u;
    const int k = __ffs((int)ge) - 8;                   // bit offset of the byte
    const int rr = r - (int)(((pre << 8) >> k) & 0xffu);
#if defined(__CUDA_ARCH__)
    const u32 t = __ldg(&lx_sel8.v[(x >> k) & 0xffu]);
#else
    const u32 t = lx_sel8.v[(x >> k) & 0xffu];
#endif
    return k + (int)((t >> (4 * rr)) & 0xfu);
}
#else
// position of the r-th (0-based) set bit of a 32-bit word; r < popc(x)
__device__ __forceinline__ int select32(u32 x, int r) {
    int pos = 0, c;
    c = __popc(x & 0xffffu);
    if (r >= c) { r -= c; x >>= 16; pos += 16; }
    c = __popc(x & 0xffu);
    if (r >= c) { r -= c; x >>= 8; pos += 8; }
    c = __popc(x & 0xfu);
    if (r >= c) { r -= c; x >>= 4; pos += 4; }
    c = __popc(x & 0x3u);
    if (r >= c) { r -= c; x >>= 2; pos += 2; }
    c = (int)(x & 1u);
    if (r >= c) { pos += 1; }
    return pos;
}
#endif

// ---- counter RNG: splitmix64 finaliser (reference rng.py:12-42) ----------
__device__ __forceinline__ u64 mix64(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
constexpr u64 HASH_SEED = 0x243F6A8885A308D3ull;

// hash_key(seed) folded once; per-ply key = mix64(seedmix ^ move_count)
__device__ __forceinline__ u64 seed_mix(u64 seed) { return mix64(HASH_SEED ^ seed); }

// r = min(int64(u * n), max(n-1, 0)) with u = (key >> 11) * 2^-53, computed in
// IEEE float64 exactly as numpy does (reference compiler.py:440-441)
// (u * n < 2^31 for every board, so the truncation and clamp stay 32-bit:
// identical values to numpy's int64 cast, one VIMNMX instead of a 64-bit
// compare and select)
__device__ __forceinline__ int draw_index(u64 key, int n) {
    const double u = __dmul_rn((double)(key >> 11), 0x1p-53);
    const int r = __double2int_rz(__dmul_rn(u, (double)n));
    const int hi = n > 1 ? n - 1 : 0;
    return r < hi ? r : hi;
}

__device__ __forceinline__ double key_uniform(u64 key) {
    return __dmul_rn((double)(key >> 11), 0x1p-53);
}

// draw_index with the uniform already formed (identical arithmetic)
__device__ __forceinline__ int draw_index_u(double u, int n) {
    const int r = __double2int_rz(__dmul_rn(u, (double)n));
    const int hi = n > 1 ? n - 1 : 0;
    return r < hi ? r : hi;
}

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }

// Per-thread shared-memory mirror of both boards, for rules that probe a few
// cells at run-time positions (anchored captures / lines on big boards): a
// probe is one LDS instead of a W-way register select, and it runs on the
// LSU pipe while the bitboard work saturates the ALU pipe.  Layout
// [word][thread] keeps every access bank-conflict free.
// Block size of the per-env kernels (lx_init / legal / sample / step /
// random_step / env_step ...): 256, or 128 for games whose per-thread
// shared-memory row mirror would not fit 48 KB of static shared memory per
// block at 256 threads (lowering: LX_BLOCK).  The per-thread shared-memory
// slots are [word][thread] with this stride.
#ifndef LX_BLOCK
#define LX_BLOCK 256
#endif
#ifndef LX_MIRROR_STRIDE
#define LX_MIRROR_STRIDE LX_BLOCK
#endif
template <int W>
struct Mirror {
    static __device__ __forceinline__ u32* slot() {
        __shared__ u32 buf[2 * W * LX_MIRROR_STRIDE];
        return buf + threadIdx.x;
    }
    // one player's plane only (readers of that plane need nothing else);
    // big boards select word by word (a selected BB<W> copy spills); small
    // boards select the board (C4: 7% faster than the word-wise form)
    static __device__ __forceinline__ void store_plane(int player, const BB<W>& p0,
                                                       const BB<W>& p1) {
        if constexpr (W <= 2) {
            const BB<W> p = player ? p1 : p0;
            u32* m = slot();
#pragma unroll
            for (int i = 0; i < W; i++) m[(player * W + i) * LX_MIRROR_STRIDE] = p.w[i];
        } else {
            u32* m = slot() + player * W * LX_MIRROR_STRIDE;
#pragma unroll
            for (int i = 0; i < W; i++) m[i * LX_MIRROR_STRIDE] = player ? p1.w[i] : p0.w[i];
        }
    }
    static __device__ __forceinline__ void store(const BB<W>& p0, const BB<W>& p1) {
        u32* m = slot();
#pragma unroll
        for (int i = 0; i < W; i++) {
            m[i * LX_MIRROR_STRIDE] = p0.w[i];
            m[(W + i) * LX_MIRROR_STRIDE] = p1.w[i];
        }
    }
    // remove `cell` from `player`'s mirrored plane (a probed capture collects
    // its cells here with LDS/LOP/STS per cell instead of a W-way register
    // select per cell; the caller diffs the plane against its registers)
    static __device__ __forceinline__ void clear(int player, int cell) {
        slot()[(player * W + (cell >> 5)) * LX_MIRROR_STRIDE] &= ~(1u << (cell & 31));
    }
    static __device__ __forceinline__ BB<W> load(int player) {
        const u32* m = slot() + player * W * LX_MIRROR_STRIDE;
        BB<W> r;
#pragma unroll
        for (int i = 0; i < W; i++) r.w[i] = m[i * LX_MIRROR_STRIDE];
        return r;
    }
    // is `cell` occupied by `player` (0/1)?
    static __device__ __forceinline__ bool probe(int player, int cell) {
        const u32 w = slot()[(player * W + (cell >> 5)) * LX_MIRROR_STRIDE];
        return (w >> (cell & 31)) & 1u;
    }
    // branch-free probe: `ok` gates a possibly off-board cell (clamped, so the
    // load stays inside the mirror)
    static __device__ __forceinline__ u32 probe_if(bool ok, int player, int cell) {
        const int c = ok ? cell : 0;
        const u32 w = slot()[(player * W + (c >> 5)) * LX_MIRROR_STRIDE];
        return ok ? ((w >> (c & 31)) & 1u) : 0u;
    }
};

// cell index of the r-th set bit (ascending cell order); r < popc(a).
// Boards of >= 6 words find the word through the shared-memory mirror slot
// (which such boards already have for their probes): each word and the
// count of set bits before it are stashed, the word index is the number of
// prefix counts <= r, and the word and its base come back with one load
// each -- 4 ALU instructions per word instead of a select chain of ~8.
template <int W>
__device__ __forceinline__ int select_bit(const BB<W>& a, int r) {
    if constexpr (W >= 6 && LX_SELECT_STASH) {
        u32* m = Mirror<W>::slot();
        int cum = 0, k = 0;
#pragma unroll
        for (int i = 0; i < W; i++) {
            m[i * LX_MIRROR_STRIDE] = a.w[i];
            m[(W + i) * LX_MIRROR_STRIDE] = (u32)cum;
            cum += __popc(a.w[i]);
            k += cum <= r;
        }
        const u32 word = m[k * LX_MIRROR_STRIDE];
        const int before = (int)m[(W + k) * LX_MIRROR_STRIDE];
        return 32 * k + select32(word, r - before);
    }
    u32 word = 0u;
    int base = 0, rem = r;
    bool found = false;
#pragma unroll
    for (int i = 0; i < W; i++) {
        const int c = __popc(a.w[i]);
        const bool here = !found && rem < c;
        word = here ? a.w[i] : word;
        base = here ? 32 * i : base;
        rem = (!found && !here) ? rem - c : rem;
        found = found || here;
    }
    return base + select32(word, rem);
}


// Per-thread row planes (generated code's rm_row / rm_build / rm_set, see
// lowering.GameLowering row mirror): NR words per player, [row][thread].
template <int NR>
struct RowMirror {
    static __device__ __forceinline__ u32* slot() {
        __shared__ u32 buf[2 * NR * LX_MIRROR_STRIDE];
        return buf + threadIdx.x;
    }
};

// position and in-ply offset of the r-th unit of a bit-sliced multiset:
// cell x carries c(x) = sum_j 2^j [x in d[j]] units, units are ordered by
// cell, and r < sum_x c(x).  Returns x; rem = r - (units of cells < x), so
// 0 <= rem < c(x).  Branch-free: word choice by prefix sums, then a 5-level
// binary descent inside the word (a slide group's "r-th (source, distance)
// pair", reference mechanics.py:211-227).
template <int W, int NB>
__device__ __forceinline__ int select_weighted(const BB<W> (&d)[NB], int r, int& rem) {
    int cum = 0, base = 0, word = 0;
    bool found = false;
#pragma unroll
    for (int i = 0; i < W; i++) {
        int c = 0;
#pragma unroll
        for (int j = 0; j < NB; j++) c += __popc(d[j].w[i]) << j;
        const bool here = !found && r < cum + c;
        word = here ? i : word;
        base = here ? cum : base;
        found = found || here;
        cum += c;
    }
    u32 v[NB];
#pragma unroll
    for (int j = 0; j < NB; j++) {
        u32 t = 0u;
#pragma unroll
        for (int i = 0; i < W; i++) t = (word == i) ? d[j].w[i] : t;
        v[j] = t;
    }
    int rr = r - base, pos = 0;
#pragma unroll
    for (int half = 16; half >= 1; half >>= 1) {
        const u32 m = ((1u << half) - 1u) << pos;
        int c = 0;
#pragma unroll
        for (int j = 0; j < NB; j++) c += __popc(v[j] & m) << j;
        const bool up = rr >= c;
        rr = up ? rr - c : rr;
        pos = up ? pos + half : pos;
    }
    rem = rr;
    return 32 * word + pos;
}

// register-resident state of one env (unpacked from the HBM state words)
template <int W, int NX, int NGC = 1>
struct State {
    BB<W> own0, own1;
    u32 ext[NX > 0 ? NX : 1];
    u32 mc;
    int cur, term, trunc, outcome, phase, pos, last_mover, last_kind, last_dest;
    int pass_streak, pf0, pf1, ldbp0, ldbp1, sc0, sc1;
    int last_source, must_move;  // movement games (reference state.py:96-104)
    int ovr, samep;              // transient per ply: extra-turn player, same-piece flag
    int ncached;                 // ntot holds the move-group totals of the position (not stored)
    int mirror_fresh;            // this ply's board planes are in the shared-memory mirror (not stored)
    int mirror_valid;            // the row mirror holds this state's planes (not stored)
    int ntot[NGC];
    u64 seed;
};

#if defined(__CUDA_ARCH__)
// ---------------------------------------------------------------------------
// Warp-cooperative flood (connectivity reach sets, reference connectivity.py
// place_update).  A sequential flood costs the warp the LONGEST flood of its
// lanes (~5.5 dilations per ply on Hex 11x11, ~54 instructions each, while
// the mean lane needs 0.4).  Here one flood is spread over a group of G lanes,
// lane i of the group holding word i of the bitboard: a dilation is 4 funnel
// shifts + 4 shuffles per lane instead of 4 words x 6 shifts, and 32/G floods
// run side by side.  The fixed point is the same set as the sequential loop.

// word i of a W-word bitboard held by one lane of a group
template <int W>
struct LW {
    u32 v;
    int i;
};
template <int W>
__device__ constexpr int lw_group() { return W <= 1 ? 1 : W <= 2 ? 2 : W <= 4 ? 4 : W <= 8 ? 8 : W <= 16 ? 16 : 32; }

template <int W>
__device__ __forceinline__ u32 word_of(const BB<W>& m, int i) {
    u32 r = m.w[0];
#pragma unroll
    for (int k = 1; k < W; k++) r = (i == k) ? m.w[k] : r;
    return r;
}
template <int W>
__device__ __forceinline__ LW<W> operator|(const LW<W>& a, const LW<W>& b) { return LW<W>{a.v | b.v, a.i}; }
template <int W>
__device__ __forceinline__ LW<W> operator&(const LW<W>& a, const LW<W>& b) { return LW<W>{a.v & b.v, a.i}; }
template <int W>
__device__ __forceinline__ LW<W> operator&(const LW<W>& a, const BB<W>& m) {
    return LW<W>{a.v & word_of<W>(m, a.i), a.i};
}

// gather (bit x = a bit (x + S)) on the lane-word view: words i+q and i+q+1
// (S > 0) or i-q and i-q-1 (S < 0) come from the group's neighbouring lanes.
// Only for walk helpers, which AND the result with the direction's validity
// mask: a masked-in bit's source cell is on the board, so the words a shuffle
// fetches from outside the group (it then returns the lane's own word) only
// reach masked-out bits and need no zeroing.
template <int W, int S>
__device__ __forceinline__ LW<W> gather(const LW<W>& a) {
    constexpr int G = lw_group<W>();
    if constexpr (S == 0) {
        return a;
    } else if constexpr (S > 0) {
        constexpr int q = S / 32;
        constexpr unsigned s = (unsigned)(S % 32);
        const u32 lo = q ? __shfl_down_sync(0xffffffffu, a.v, q, G) : a.v;
        u32 r = lo;
        if constexpr (s != 0) {
            const u32 hi = __shfl_down_sync(0xffffffffu, a.v, q + 1, G);
            r = __funnelshift_r(lo, hi, s);
        }
        return LW<W>{r, a.i};
    } else {
        constexpr int q = (-S) / 32;
        constexpr unsigned s = (unsigned)((-S) % 32);
        const u32 hi = q ? __shfl_up_sync(0xffffffffu, a.v, q, G) : a.v;
        u32 r = hi;
        if constexpr (s != 0) {
            const u32 lo = __shfl_up_sync(0xffffffffu, a.v, q + 1, G);
            r = __funnelshift_l(lo, hi, s);
        }
        return LW<W>{r, a.i};
    }
}

__device__ __forceinline__ int lane_id() {
    u32 l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return (int)l;
}

// All 32 lanes call this (the caller checks __activemask() == full).  Lanes
// with `need` get f = the component of f's cells inside `free_` (f ⊆ free_):
// the fixed point of f <- (f | dil(f)) & free_.  Floods are handed to lane
// groups in lane order, 32/G per round; the words travel through a per-warp
// shared-memory slot row (word k of the r-th flood at slot r*G + k, so each
// lane reads its own slot), which keeps the hand-off off the ALU pipe.
template <int W, class Dil>
__device__ __forceinline__ void coop_flood(bool need, const BB<W>& free_, BB<W>& f, Dil dil) {
    constexpr int G = lw_group<W>();
    constexpr int NGRP = 32 / G;
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ u32 lx_flood_buf[32][2][32];        // [warp of the block][free|f][slot]
    const int lane = lane_id();
    u32 (&buf)[2][32] = lx_flood_buf[(threadIdx.x >> 5) & 31];
    const int grp = lane / G, idx = lane % G;
    unsigned pending = __ballot_sync(FULL, need);
    while (pending) {
        const int rank = __popc(pending & ((1u << lane) - 1u));
        const bool mine = ((pending >> lane) & 1u) && rank < NGRP;
        __syncwarp(FULL);
        if (mine) {
#pragma unroll
            for (int k = 0; k < W; k++) {
                buf[0][rank * G + k] = free_.w[k];
                buf[1][rank * G + k] = f.w[k];
            }
        }
        __syncwarp(FULL);
        const bool act = grp < __popc(pending) && idx < W;
        LW<W> x{act ? buf[1][lane] : 0u, idx};
        const LW<W> fre{act ? buf[0][lane] : 0u, idx};
        while (true) {
            const LW<W> g = (x | dil(x)) & fre;
            const bool ch = g.v != x.v;
            x = g;
            if (!__any_sync(FULL, ch)) break;
        }
        __syncwarp(FULL);
        buf[1][lane] = x.v;
        __syncwarp(FULL);
        if (mine) {
#pragma unroll
            for (int k = 0; k < W; k++) f.w[k] = buf[1][rank * G + k];
        }
        pending &= ~__ballot_sync(FULL, mine);
    }
}
#endif

}  // namespace lx
