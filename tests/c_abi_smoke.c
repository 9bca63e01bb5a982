/* c_abi_smoke.c -- TEST INFRASTRUCTURE: a plain C caller of the backend,
 * using nothing but include/ludax_b200.h (and the CUDA runtime for device
 * memory).  Every buffer is sized from lx_game_info alone:
 *   bind device -> create -> info -> init -> fused rollout -> export
 * and the exported reference-layout arrays are written to a file that
 * tests/test_c_abi.py compares with the CPU oracle; then the same episode
 * once more through lx_playout_host with host buffers only.
 *
 *   c_abi_smoke <lowered.cu> <name> <include_dir> <cache_dir> <B> <seed> <out.bin>
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "ludax_b200.h"

#define CHECK(call)                                                                      \
    do {                                                                                 \
        int st_ = (call);                                                                \
        if (st_ != LX_OK) {                                                              \
            fprintf(stderr, "%s failed: %d %s\n", #call, st_, lx_last_error());          \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

static void *dalloc(size_t n) {
    void *p = NULL;
    if (cudaMalloc(&p, n ? n : 1) != cudaSuccess) {
        fprintf(stderr, "cudaMalloc(%zu) failed\n", n);
        exit(1);
    }
    cudaMemset(p, 0, n ? n : 1);
    return p;
}

static int dump(FILE *f, const char *name, const void *dev, size_t n) {
    void *h = malloc(n ? n : 1);
    if (cudaMemcpy(h, dev, n, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    unsigned long long len = n;
    fprintf(f, "%s\n", name);
    fwrite(&len, sizeof(len), 1, f);
    fwrite(h, 1, n, f);
    free(h);
    return 0;
}

int main(int argc, char **argv) {
    if (argc != 8) {
        fprintf(stderr, "usage: %s lowered.cu name include_dir cache_dir B seed out.bin\n", argv[0]);
        return 2;
    }
    FILE *sf = fopen(argv[1], "rb");
    if (!sf) return 2;
    fseek(sf, 0, SEEK_END);
    long sn = ftell(sf);
    fseek(sf, 0, SEEK_SET);
    char *src = (char *)calloc((size_t)sn + 1, 1);
    if (fread(src, 1, (size_t)sn, sf) != (size_t)sn) return 2;
    fclose(sf);
    const int64_t B = atoll(argv[5]);
    const uint64_t seed = strtoull(argv[6], NULL, 10);

    CHECK(lx_bind_device(0));
    lx_game *g = NULL;
    CHECK(lx_game_create(src, argv[2], argv[3], argv[4], &g));
    lx_game_info info;
    CHECK(lx_game_info_get(g, &info));
    printf("info C=%d A=%d pass=%d W=%d NQ=%d state_bytes=%d NX=%d mech=%d mask_words=%d "
           "device=%d sms=%d blocks=%d threads=%d\n",
           info.num_cells, info.num_actions, info.pass_index, info.board_words, info.state_quads,
           info.state_bytes, info.private_words, info.mechanics, info.mask_words, info.device,
           info.num_sms, info.rollout_blocks, info.rollout_threads);
    if (info.num_cells <= 0 || info.num_actions < info.num_cells || info.state_quads <= 0 ||
        info.state_bytes != 16 * info.state_quads || info.board_words * 32 < info.num_cells) {
        fprintf(stderr, "lx_game_info is not populated\n");
        return 3;
    }
    const int64_t C = info.num_cells;

    void *state = dalloc((size_t)B * (size_t)info.state_bytes);
    uint64_t *stats = (uint64_t *)dalloc(8 * sizeof(uint64_t));
    void *work = dalloc(LX_ROLLOUT_WORK_BYTES);   /* zero-filled once; every call leaves it zeroed */
    CHECK(lx_init(g, state, B, NULL, seed, 0, NULL));
    /* continue the initialised envs (mode 0), store finals (2), truncate at the cap (4) */
    int64_t stuck = -1;
    CHECK(lx_rollout(g, state, B, 200, 2 | 4, 0, NULL, 0, stats, work, NULL, NULL, 1, &stuck,
                     NULL));

    lx_ref_state ref;
    memset(&ref, 0, sizeof(ref));
    ref.board_piece = (int8_t *)dalloc((size_t)(B * C));
    ref.board_owner = (int8_t *)dalloc((size_t)(B * C));
    ref.current_player = (int8_t *)dalloc((size_t)B);
    ref.move_count = (int32_t *)dalloc((size_t)B * 4);
    ref.terminated = (uint8_t *)dalloc((size_t)B);
    ref.truncated = (uint8_t *)dalloc((size_t)B);
    ref.outcome = (int8_t *)dalloc((size_t)B);
    ref.seeds = (uint64_t *)dalloc((size_t)B * 8);
    CHECK(lx_export(g, state, B, &ref, NULL));
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;

    uint64_t hs[8];
    cudaMemcpy(hs, stats, sizeof(hs), cudaMemcpyDeviceToHost);
    printf("stats steps=%llu p1=%llu p2=%llu draws=%llu truncated=%llu envs=%llu\n",
           (unsigned long long)hs[0], (unsigned long long)hs[1], (unsigned long long)hs[2],
           (unsigned long long)hs[3], (unsigned long long)hs[4], (unsigned long long)hs[5]);

    FILE *f = fopen(argv[7], "wb");
    if (!f) return 5;
    int bad = 0;
    bad |= dump(f, "board_piece", ref.board_piece, (size_t)(B * C));
    bad |= dump(f, "board_owner", ref.board_owner, (size_t)(B * C));
    bad |= dump(f, "current_player", ref.current_player, (size_t)B);
    bad |= dump(f, "move_count", ref.move_count, (size_t)B * 4);
    bad |= dump(f, "terminated", ref.terminated, (size_t)B);
    bad |= dump(f, "truncated", ref.truncated, (size_t)B);
    bad |= dump(f, "outcome", ref.outcome, (size_t)B);
    bad |= dump(f, "seeds", ref.seeds, (size_t)B * 8);
    bad |= dump(f, "stats", stats, 8 * sizeof(uint64_t));
    fclose(f);

    /* the same episode through the host-buffer call: no device memory on the
       caller's side at all (seeds spawned from `seed`, outcomes / move counts /
       stats written to host arrays) */
    int8_t *h_out = (int8_t *)malloc((size_t)B);
    int32_t *h_turns = (int32_t *)malloc((size_t)B * 4);
    uint64_t h_stats[8];
    CHECK(lx_playout_host(g, B, 200, LX_PLAYOUT_TRUNCATE, seed, NULL, 0, h_out, h_turns, h_stats,
                          NULL, &stuck, NULL));
    f = fopen(argv[7], "ab");
    if (!f) return 5;
    unsigned long long len = (unsigned long long)B;
    fprintf(f, "host_outcome\n");
    fwrite(&len, sizeof(len), 1, f);
    fwrite(h_out, 1, (size_t)B, f);
    len = (unsigned long long)B * 4;
    fprintf(f, "host_move_count\n");
    fwrite(&len, sizeof(len), 1, f);
    fwrite(h_turns, 1, (size_t)B * 4, f);
    len = sizeof(h_stats);
    fprintf(f, "host_stats\n");
    fwrite(&len, sizeof(len), 1, f);
    fwrite(h_stats, 1, sizeof(h_stats), f);
    fclose(f);
    free(h_out);
    free(h_turns);
    CHECK(lx_game_destroy(g));
    return bad ? 6 : 0;
}
