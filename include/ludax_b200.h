/*
 * ludax_b200.h -- C-ABI of the B200 game-simulation backend.
 *
 * Replaces the reference's numpy runtime behind CompiledGame / engine
 * (reference: pkg/src/boardlang/compiler.py:197-650, engine.py:27-163).
 * Plain C types only: device pointers are `void*` / typed pointers into
 * CUDA global memory (e.g. torch tensors' data_ptr()), streams are CUstream
 * handles passed as `void*` (NULL = legacy default stream).  No C++
 * exceptions cross this boundary; every entry point returns an LX_* status
 * and lx_last_error() describes the last failure on the calling thread.
 *
 * One game = one handle = one NVRTC-compiled sm_100a module.  Handles are
 * immutable after creation and may be shared across threads and streams;
 * the library keeps no pointer to caller memory past a call.
 */
#ifndef LUDAX_B200_H
#define LUDAX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python shim re-raises them as the reference exception
   types (reference errors.py:59-76) */
#define LX_OK 0
#define LX_EILLEGAL_ACTION 1   /* IllegalAction   (mechanics.py:503-510, compiler.py:484-494) */
#define LX_ETERMINAL_STATE 2   /* TerminalState   (engine.py:31-33, 43-44) */
#define LX_EEMPTY_MASK 3       /* EmptyMask       (engine.py:142-147) */
#define LX_ECOMPILE 4          /* CompileError    (errors.py:71-76), NVRTC stage */
#define LX_ECUDA 5             /* driver / launch failure */
#define LX_EINVALID 6          /* bad argument */

typedef struct lx_game lx_game;

/* Static facts of a compiled game (reference CompiledGame.describe,
   compiler.py:628-650, plus the device state layout), read from the
   generated unit's lx_facts constant at lx_game_create: a C caller sizes
   every buffer from these alone. */
typedef struct {
    int32_t num_cells;          /* C */
    int32_t num_actions;        /* A: C, C*C (movement) or #directions (gridworld), +1 pass; ActionCodec.size (codec.py:58-69) */
    int32_t pass_index;         /* -1 when the game has no pass action */
    int32_t board_words;        /* W: 32-bit words per player bitboard */
    int32_t state_quads;        /* NQ: 16-byte quads per env in HBM; a batch of B envs is NQ*B*16 bytes */
    int32_t state_bytes;        /* 16 * NQ: device bytes per env */
    int32_t private_words;      /* NX: piece-type planes + rule-private words per env */
    int32_t mechanics;          /* 0 placement, 1 movement, 2 gridworld */
    int32_t mask_words;         /* ceil(A / 32): u32 words per bit-packed mask row */
    int32_t device;             /* CUDA device ordinal the handle is bound to */
    int32_t num_sms;            /* SMs of that device */
    int32_t rollout_blocks;     /* persistent grid of lx_rollout (SMs x blocks/SM) */
    int32_t rollout_threads;    /* block size of lx_rollout */
} lx_game_info;

/* Reference GameState field pointers (state.py:78-130); optional fields NULL.
   Used by lx_export / lx_import to move between the device bitboard layout
   and the reference's int8 cell arrays. */
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
    int16_t *must_move;         /* movement games with same-piece extra turns */
    int8_t *turn_pos;           /* orders with a repeated player */
    uint8_t *hopped_mask, *captured_mask, *promoted_mask;   /* (B, C) transient masks */
} lx_ref_state;

int lx_version(void);
const char *lx_last_error(void);

/* Compile (or fetch from cache_dir) the generated translation unit and load
   it on the calling thread's current CUDA context (the device selected with
   cudaSetDevice / torch.cuda.set_device / lx_bind_device; no current context
   is an LX_ECUDA error).  The handle is bound to that device: calls made
   while another device is current fail with LX_EINVALID -- create one handle
   per device.  Replaces CompiledGame.__init__ (compiler.py:200-286).
   `source` is the lowering's output; headers are resolved from include_dir;
   cubins are cached as <cache_dir>/<key>-g<group>.cubin. */
int lx_game_create(const char *source, const char *name, const char *include_dir,
                   const char *cache_dir, lx_game **out);
/* Make device `ordinal`'s primary context current on the calling thread
   (for C callers that do not use the CUDA runtime). */
int lx_bind_device(int ordinal);
/* Compile to <cache_dir>/<key>.cubin only (no GPU needed); *key_out gets the
   cache key (>= 65 bytes). */
int lx_compile_only(const char *source, const char *name, const char *include_dir,
                    const char *cache_dir, char *key_out);
/* Cache key of (source, headers in include_dir, NVRTC options) without
   compiling (>= 65 bytes). */
int lx_cache_key(const char *source, const char *include_dir, char *key_out);
int lx_game_info_get(const lx_game *g, lx_game_info *out);
int lx_game_destroy(lx_game *g);

/* CompiledGame.init (compiler.py:357-364): seeds[i], or when seeds is NULL
   spawn_seeds: hash_key(seed, first_index + i) (rng.py:52-54). */
int lx_init(const lx_game *g, void *state, int64_t B, const uint64_t *seeds, uint64_t seed,
            int64_t first_index, void *stream);

/* CompiledGame.legal_mask / legal_counts (compiler.py:394-428):
   mask (B, A) uint8 or NULL, counts (B,) int64 or NULL; mover (B,) int8 or
   NULL: legality for that player instead of each row's current player (the
   reference's `mover=` argument), in the row's own phase. */
int lx_legal(const lx_game *g, const void *state, int64_t B, const int8_t *mover, uint8_t *mask,
             int64_t *counts, void *stream);

/* CompiledGame.sample_actions (compiler.py:430-446): u (B,) float64 draws, or
   NULL to draw uniform(seed, move_count) on device (engine.random_actions);
   mover as in lx_legal. */
int lx_sample(const lx_game *g, const void *state, int64_t B, const int8_t *mover, const double *u,
              int64_t *actions, void *stream);

/* Mark rows (B,) uint8 (NULL = all) that are still live terminated +
   truncated draws in place (engine.playout_random's cap, engine.py:156-160;
   agents.py:430-435). */
int lx_truncate(const lx_game *g, void *state, int64_t B, const uint8_t *rows, void *stream);

/* Replace every row's RNG seed with seeds (B,) uint64 (device) in place
   (the MCTS rollout re-keying, agents.py:229-233). */
int lx_set_seeds(const lx_game *g, void *state, int64_t B, const uint64_t *seeds, void *stream);

/* CompiledGame.step_into (compiler.py:456-580), in place on rows (B,) uint8
   (NULL = all) & ~terminated.  verify != 0 checks every live row first and
   fails with LX_EILLEGAL_ACTION (*bad_row = first bad row) before mutating;
   scratch is >= 8 bytes of device memory (used only when verifying). */
int lx_step(const lx_game *g, void *state, int64_t B, const int64_t *actions,
            const uint8_t *rows, int verify, void *scratch, int64_t *bad_row, void *stream);

/* One fused ply of uniform-random play for rows with !terminated and
   move_count < max_turns (engine.random_actions + step_into); actions_out
   (B,) int64 or NULL receives the sampled actions (-1 for idle rows). */
int lx_random_step(const lx_game *g, void *state, int64_t B, int max_turns,
                   int64_t *actions_out, void *stream);

/* MCTS expansion with rollouts (agents._Search._attach_and_rollout and
   agents._rollout, agents.py:211-238, 313-353), one thread per child: in a
   node pool of `cap` env rows, child row children[i] = parent row parents[i]
   stepped with actions[i]; info[i] = current_player | terminated << 2 |
   (outcome + 1) << 3 | legal_count << 8; masks (n, A) uint8 or NULL gets the
   child's legal mask; rolled[i] = outcome of one uniform-random rollout from
   a live child with legal actions, drawing with seeds[i] and capped at
   max_turns total plies (0 draw / cap / stuck, 1 P1, 2 P2), else -1.
   All pointers are device memory. */
int lx_expand(const lx_game *g, void *pool, int64_t cap, const int64_t *parents,
              const int64_t *actions, const int64_t *children, int64_t n, const uint64_t *seeds,
              int max_turns, int32_t *info, int8_t *rolled, uint8_t *masks, void *stream);

/* One UCB1 MCTS decision per root state (agents._Search.run, agents.py:84-310:
   forced prefix, iterations of selection / expansion / rollout / backprop,
   best child), one warp per tree: the lanes split each node's UCB1 scores and
   the action-order sort; the rest runs on identical data in every lane.
   keys[t] = the tree key, budgets[t] = iterations; logs[N] = log(N) as the
   host computes it (N < nlogs); arena: n * arena_bytes bytes (node records,
   action and child lists, a sort scratch of 12 * (A + 1) bytes); pool:
   pool_rows >= n * nmax env rows (node states).  shared_bytes > 0: each
   tree's arena (arena_bytes) and its node states (nmax * 16 * NQ) live in
   that much dynamic shared memory instead (<= the device's opt-in limit;
   arena / pool are then unused).  actions_out[t] = chosen action (-1:
   none); status[t] = 1 when a capacity was exceeded (the caller searches on
   the host instead).  Device memory throughout. */
int lx_mcts(const lx_game *g, const void *roots, int64_t n, const uint64_t *keys,
            const int32_t *budgets, double exploration, int rollout_max_turns, const double *logs,
            int32_t nlogs, void *pool, int64_t pool_rows, int32_t nmax, void *arena,
            int64_t arena_bytes, int64_t *actions_out, int32_t *status, int32_t shared_bytes,
            void *stream);

/* Fused register-resident rollout (engine.playout_random, engine.py:123-163;
   evaluation._run_episode, evaluation.py:197-211).  One kernel launch, no
   memsets:
   mode bit 0: start envs from seeds (seeds[i] or spawn(seed, first_index+i))
                 else continue from `state`
   mode bit 1: write final states to `state`
   mode bit 2: mark unfinished envs terminated+truncated draws at max_turns
   mode bit 3 (LX_ROLLOUT_CLEAR_WORK): zero `work` first (one memset)
   work: LX_ROLLOUT_WORK_BYTES of device scratch, zero-filled before its first
   use; every call leaves it zeroed again (the last block clears it), so
   reusing one buffer per stream needs no clearing.
   stats: u64[8] device buffer, written: steps, p1 wins, p2 wins, draws,
   truncated, envs, lowest stuck row (~0 = none), 0.  outcomes (B,) int8 /
   turns (B,) int32, or NULL: per-env outcome (0 draw, 1 P1, 2 P2) and final
   move_count.  stuck rows -> LX_EEMPTY_MASK only when check != 0 (syncs). */
#define LX_ROLLOUT_CLEAR_WORK 8
#define LX_ROLLOUT_WORK_BYTES 128
int lx_rollout(const lx_game *g, void *state, int64_t B, int max_turns, int mode, uint64_t seed,
               const uint64_t *seeds, int64_t first_index, uint64_t *stats, void *work,
               int8_t *outcomes, int32_t *turns, int check, int64_t *stuck_row, void *stream);

/* One batch episode with HOST buffers: what a numpy / ctypes caller of the
   reference's random-play loop binds (evaluation._run_episode,
   evaluation.py:197-211: init(batch, seed) then play to the end; and
   engine.playout_random, engine.py:123-163: its outcomes and move counts).
   Envs start from seeds[i] (host (B,) uint64, e.g. spawn_seeds(seed, B)) or,
   when seeds is NULL, from spawn(seed, first_index + i).  Host outputs, any
   but stats may be NULL: outcomes (B,) int8 (0 draw, 1 P1, 2 P2), turns (B,)
   int32 final move_count, stats u64[8] as lx_rollout's.  state (device,
   NQ*16*B bytes, or NULL) receives the final states.  flags:
     LX_PLAYOUT_TRUNCATE     envs reaching max_turns end as truncated draws
                             (engine.py:156-160); without it they stop there
                             unfinished (_run_episode)
     LX_PLAYOUT_UPLOAD_FIRST copy all seeds to device memory before the launch
                             (no streaming, no zero copy)
   The handle owns the device scratch (grown to the largest B seen; calls on
   one handle serialize).  Batches of >= LX_PLAYOUT_STREAM_MIN envs stream
   their seeds up in <= 64 pieces on a copy stream while the rollout already
   plays (each warp waits only for its chunk's piece), so the upload overlaps
   the play; batches of <= LX_PLAYOUT_ZERO_COPY_MAX envs use no DMA at all
   (the kernel reads the seeds from and writes its outputs to a mapped pinned
   block of the handle).  The call returns once the outputs are in host
   memory.  Pinned
   host memory (cudaHostAlloc / torch pin_memory) gets full PCIe bandwidth;
   pageable memory works without the overlap.  A live env with no legal
   action and no pass -> LX_EEMPTY_MASK (*stuck_row = lowest such env), the
   outputs still written (engine.py:142-147). */
#define LX_PLAYOUT_TRUNCATE 1
#define LX_PLAYOUT_UPLOAD_FIRST 2
#define LX_PLAYOUT_STREAM_MIN 65536
#define LX_PLAYOUT_ZERO_COPY_MAX 8192
int lx_playout_host(const lx_game *g, int64_t B, int max_turns, int flags, uint64_t seed,
                    const uint64_t *seeds, int64_t first_index, int8_t *outcomes,
                    int32_t *turns, uint64_t *stats, void *state, int64_t *stuck_row,
                    void *stream);

/* lx_playout_host split in two for callers that play many episodes back to
   back (the reference's benchmark_throughput loop, evaluation.py:214-233):
   _async enqueues the episode and returns a ticket at once; _wait returns
   when that episode's outputs are in host memory (LX_EEMPTY_MASK as above).
   Episodes alternate between two device slots of the handle: episode i+1's
   seed upload (its own stream) and episode i-1's download (a third stream)
   overlap episode i's rollout on `stream`; reuse of a slot is ordered on
   the GPU (an upload waits for the rollout two back, a rollout for the
   download two back), so _async never blocks the host (except to grow a
   slot).  Batches of <= LX_PLAYOUT_ZERO_COPY_MAX envs use no DMA (a mapped
   pinned block per slot, as lx_playout_host; the outputs reach the caller's
   buffers at _wait, or when the slot is reused).  Host buffers must stay
   valid until their ticket completes and should be pinned (pageable copies
   serialise with the rollout).  Calls on one handle serialize. */
int lx_playout_host_async(const lx_game *g, int64_t B, int max_turns, int flags, uint64_t seed,
                          const uint64_t *seeds, int64_t first_index, int8_t *outcomes,
                          int32_t *turns, uint64_t *stats, void *state, void *stream,
                          int64_t *ticket);
int lx_playout_host_wait(const lx_game *g, int64_t ticket, int64_t *stuck_row);

/* PGX-style environment step (LudaxEnvironment.step; BASELINE north star),
   one launch per ply.  flags (LX_ENV_*):
     STEP       apply one ply to live rows (else only refresh the outputs)
     RANDOM     sample a uniform legal action per live row from its own
                (seed, move_count) stream in the kernel (engine.random_actions,
                engine.py:72-75); written to `actions` when non-NULL.  Without
                RANDOM, actions (B,) int64 are read.
     AUTO_RESET re-initialise finished rows with seed hash_key(seed, 0xE9)
                (engine.reset_rows, engine.py:58-65); the terminating ply's
                terminated / truncated / rewards are still reported
     MASK_BITS  mask is (B, ceil(A/32)) uint32 bit rows (action a = bit a%32
                of word a/32) instead of (B, A) uint8
   rewards (B, 2) float32: the terminating ply's outcome (engine.py:79-87),
   0 otherwise; games reaching max_turns (> 0) end as truncated draws.  An
   illegal given action (engine.step -> IllegalAction, mechanics.py:503-510)
   is not applied: the row terminates with the PGX penalty (mover -1,
   opponent +1, outcome = opponent win); a RANDOM row with no legal action
   and no pass (EmptyMask, engine.py:142-147) ends as a truncated draw.
   Either way *bad_row (device int64, or NULL) receives the lowest such row,
   -1 when none.  Then the next state's legal mask, terminated / truncated
   (B,) uint8 and current player (B,) int32 are written.  Any output may be
   NULL. */
#define LX_ENV_AUTO_RESET 1
#define LX_ENV_RANDOM 2
#define LX_ENV_MASK_BITS 4
#define LX_ENV_STEP 8
int lx_env_step(const lx_game *g, void *state, int64_t B, int64_t *actions, int max_turns,
                int flags, void *mask, float *rewards, uint8_t *terminated, uint8_t *truncated,
                int32_t *player, int64_t *bad_row, void *stream);

/* device state <-> reference GameState arrays (device pointers).  Export:
   board_owner / board_piece may both be NULL (scalar fields only); any
   other field NULL is skipped. */
int lx_export(const lx_game *g, const void *state, int64_t B, const lx_ref_state *ref,
              void *stream);
int lx_import(const lx_game *g, void *state, int64_t B, const lx_ref_state *ref, void *stream);

/* CompiledGame.observe planes (compiler.py:611-626): (B, 3, C) uint8 */
int lx_observe(const lx_game *g, const void *state, int64_t B, int player, uint8_t *planes,
               void *stream);

#ifdef __cplusplus
}
#endif
#endif
