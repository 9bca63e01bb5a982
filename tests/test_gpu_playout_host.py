"""lx_playout_host: one batch episode with host buffers (the reference's
_run_episode / playout_random as a numpy caller binds them,
evaluation.py:197-211, engine.py:123-163).  Checked against the CPU oracle
and against the device-buffer lx_rollout on the same seeds, with the seeds
streamed (>= LX_PLAYOUT_STREAM_MIN envs) and uploaded first.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2506_22609_b200 as lx  # noqa: E402
from oracle import oracle as O  # noqa: E402

STREAM_MIN = 65536          # LX_PLAYOUT_STREAM_MIN (include/ludax_b200.h)
_G = {}


def game(name):
    if name not in _G:
        _G[name] = lx.load_config_game(name)
    return _G[name]


def device_rollout(g, seeds, truncate=True, max_turns=200):
    B = len(seeds)
    out = torch.empty(B, dtype=torch.int8, device="cuda")
    turns = torch.empty(B, dtype=torch.int32, device="cuda")
    _, st = g.rollout(seeds=seeds, store=False, truncate=truncate, max_turns=max_turns,
                      outcomes=out, turns=turns)
    return out.cpu().numpy(), turns.cpu().numpy(), st.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("name,B", [("tic_tac_toe", 1000), ("connect_four", 200_003),
                                    ("hex", 70_001), ("reversi", 4096), ("pente", 65_536)])
def test_host_call_matches_oracle_and_device_rollout(name, B):
    g = game(name)
    seeds = O.spawn_seeds(77, B)
    outc, turns, stats = g.playout_host(seeds=seeds, turns=True)
    d_out, d_turns, d_stats = device_rollout(g, seeds)
    assert np.array_equal(outc, d_out) and np.array_equal(turns, d_turns)
    assert np.array_equal(stats[:6], d_stats[:6])
    assert stats[6] == np.uint64(2 ** 64 - 1) and stats[7] == 0
    assert int(stats[0]) == int(turns.astype(np.int64).sum())
    W = min(B, 2048 if name in ("tic_tac_toe", "connect_four") else 256)
    for off in (0, B - W):                 # head and tail windows vs the oracle
        want, _ = O.OracleGame(name).playout(seeds=seeds[off:off + W], threads=8)
        assert np.array_equal(outc[off:off + W], want["outcome"]), (name, off)
        assert np.array_equal(turns[off:off + W], want["move_count"]), (name, off)


def test_streamed_equals_upload_first_and_pinned_equals_pageable():
    g = game("connect_four")
    B = 3 * STREAM_MIN + 17
    seeds = O.spawn_seeds(5, B)
    a = g.playout_host(seeds=seeds, turns=True)
    b = g.playout_host(seeds=seeds, turns=True, upload_first=True)
    pinned = torch.from_numpy(seeds.view(np.int64)).pin_memory()
    o_p = torch.empty(B, dtype=torch.int8).pin_memory()
    t_p = torch.empty(B, dtype=torch.int32).pin_memory()
    s_p = torch.empty(8, dtype=torch.int64).pin_memory()
    g.playout_host(seeds=pinned, outcomes=o_p, turns=t_p, stats=s_p)
    for x in (b, (o_p.numpy(), t_p.numpy(), s_p.numpy().view(np.uint64))):
        assert np.array_equal(a[0], x[0]) and np.array_equal(a[1], x[1])
        assert np.array_equal(a[2], x[2])


def test_spawned_seeds_first_index_and_final_states():
    g = game("connect_four")
    B, first = 100_000, 12345
    outc, turns, stats = g.playout_host(batch_size=B, seed=9, first_index=first, turns=True,
                                        out=g.empty_state(B))
    d_out, d_turns, _ = device_rollout(g, O.spawn_seeds(9, B, first=first))
    assert np.array_equal(outc, d_out) and np.array_equal(turns, d_turns)
    st = g.empty_state(B)
    g.playout_host(seeds=O.spawn_seeds(9, B, first=first), outcomes=False, out=st)
    ref, _ = g.rollout(seeds=O.spawn_seeds(9, B, first=first), out=g.empty_state(B))
    assert st.digest() == ref.digest()


def test_untruncated_cap_and_repeated_calls_reuse_scratch():
    g = game("pente")
    seeds = O.spawn_seeds(3, 4096)
    # the cap without truncation leaves unfinished envs (_run_episode)
    o1, t1, s1 = g.playout_host(seeds=seeds, max_turns=40, truncate=False, turns=True)
    d_out, d_turns, d_stats = device_rollout(g, seeds, truncate=False, max_turns=40)
    assert np.array_equal(o1, d_out) and np.array_equal(t1, d_turns)
    assert np.array_equal(s1[:6], d_stats[:6])
    assert int(t1.max()) == 40 and int(s1[4]) == 0
    for B in (STREAM_MIN * 2, 33, STREAM_MIN * 2):        # shrink and regrow
        s = O.spawn_seeds(11, B)
        o, t, _ = g.playout_host(seeds=s, turns=True)
        d_o, d_t, _ = device_rollout(g, s)
        assert np.array_equal(o, d_o) and np.array_equal(t, d_t)


def test_empty_batch_and_bad_arguments():
    g = game("tic_tac_toe")
    outc, turns, stats = g.playout_host(seeds=np.zeros(0, dtype=np.uint64))
    assert outc.size == 0 and stats[:6].tolist() == [0] * 6
    assert stats[6] == np.uint64(2 ** 64 - 1)
    with pytest.raises(ValueError):
        g.playout_host(seeds=np.zeros(10, dtype=np.uint64), outcomes=np.zeros(9, np.int8))


@pytest.mark.parametrize("B", [1, 31, 256, 257, 1000, 2048, 2049, 5000])
def test_small_grids_one_block_cluster_and_ticket_publish(B):
    """Batch sizes across the three stats-publish paths of lx_rollout (one
    block, one cluster of 2..8 blocks, cross-block ticket): outcomes, move
    counts and stats equal the oracle's."""
    g = game("connect_four")
    seeds = O.spawn_seeds(2718, B)
    d_out, d_turns, d_stats = device_rollout(g, seeds)
    want, steps = O.OracleGame("connect_four").playout(seeds=seeds, threads=8)
    assert np.array_equal(d_out, want["outcome"]) and np.array_equal(d_turns, want["move_count"])
    assert int(d_stats[0]) == steps and int(d_stats[5]) == B
    assert int(d_stats[1] + d_stats[2] + d_stats[3]) == B
    assert d_stats[6] == np.uint64(2 ** 64 - 1) and d_stats[7] == 0
    h_out, h_turns, h_stats = g.playout_host(seeds=seeds, turns=True)
    assert np.array_equal(h_out, d_out) and np.array_equal(h_stats, d_stats)
    assert np.array_equal(h_turns, d_turns)
    # zero-copy (B <= LX_PLAYOUT_ZERO_COPY_MAX) and the device-copy path agree
    u_out, u_turns, u_stats = g.playout_host(seeds=seeds, turns=True, upload_first=True)
    assert np.array_equal(u_out, d_out) and np.array_equal(u_turns, d_turns)
    assert np.array_equal(u_stats, d_stats)


def test_async_pipeline_matches_sync_calls():
    """lx_playout_host_async / _wait with two episodes in flight equals the
    synchronous call episode by episode (slot reuse, tickets in order and out
    of order, an empty batch in the stream of calls)."""
    g = game("connect_four")
    sizes = [STREAM_MIN * 2, 5000, 0, STREAM_MIN * 2 + 1, 1]
    seeds = [O.spawn_seeds(100 + k, B) for k, B in enumerate(sizes)]
    pinned = [torch.from_numpy(s.view(np.int64)).pin_memory() for s in seeds]
    outs = [torch.empty(B, dtype=torch.int8).pin_memory() for B in sizes]
    turns = [torch.empty(B, dtype=torch.int32).pin_memory() for B in sizes]
    stats = [torch.zeros(8, dtype=torch.int64).pin_memory() for _ in sizes]
    tickets = []
    for k in range(len(sizes)):
        tickets.append(g.playout_host_async(seeds=pinned[k], outcomes=outs[k], turns=turns[k],
                                            stats=stats[k]))
    for t in reversed(tickets):             # waiting out of order is fine
        g.playout_host_wait(t)
    for k, B in enumerate(sizes):
        o, tn, st = g.playout_host(seeds=seeds[k], turns=True)
        assert np.array_equal(outs[k].numpy(), o) and np.array_equal(turns[k].numpy(), tn)
        assert np.array_equal(stats[k].numpy().view(np.uint64), st), k


# Test program: only the bottom row of a 3x3 board takes stones and no line
# can form there (P1, P2, P1), so every env is stuck at ply 3 with no pass.
STUCK = """(game "StuckAtThree"
  (players 2)
  (equipment
    (board (square 3))
    (pieces ("stone" both)))
  (rules
    (play
      (repeat (P1 P2)
        (place "stone"
          (destination (and (empty) (edge bottom))))))
    (end
      (if (line "stone" 3) (mover win)))))"""


@pytest.mark.parametrize("B", [100, STREAM_MIN + 5])
def test_stuck_rows_raise_empty_mask_naming_the_lowest_row(B):
    """A live env with no legal action and no pass is EmptyMask
    (engine.py:142-147) on every host-buffer path, with the lowest such row."""
    from paper_2506_22609_b200.errors import EmptyMask
    g = lx.load_game(STUCK)
    with pytest.raises(EmptyMask, match=r"\b0\b"):
        g.playout_host(batch_size=B, seed=1)
    seeds = O.spawn_seeds(1, B)
    with pytest.raises(EmptyMask):
        g.playout_host(seeds=seeds, turns=True)
    t = g.playout_host_async(seeds=torch.from_numpy(seeds.view(np.int64)).pin_memory())
    with pytest.raises(EmptyMask):
        g.playout_host_wait(t)
