"""Multi-GPU host logic on CPU: world_size-2 gloo process group.

The env path shards with no data-path collective; these tests check the sharding arithmetic,
that virtual shards of the oracle reproduce one unsharded run byte for byte (trajectories are
keyed by global env id), and the counter all_reduce / max-over-ranks timing over gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import helpers as H
from paper_1907_08467_b200 import dist as D
from paper_1907_08467_b200.inputs import games


def test_shard_arithmetic():
    assert D.shard(32768, 3) == (98304, 32768)
    parts = [D.shard_total(1001, r, 4) for r in range(4)]
    assert sum(c for _, c in parts) == 1001
    assert [b for b, _ in parts] == [0, 251, 501, 751]


def test_virtual_shards_equal_unsharded(orc):
    """G shards run one after another with env_index_base = k*N/G reproduce one N-env run."""
    roms = [games.build_rom("R1"), games.build_rom("R2")]
    N, G, steps = 8, 4, 12
    acts = H.random_actions(N, steps, 31)
    full = orc.OracleEnv(roms, N, 4, H.palette_rgb(), reset_cache_size=4)
    full.reset(2)
    ref = [full.step(acts[t]) for t in range(steps)]
    tot = np.zeros(4, np.int64)
    for k in range(G):
        base, n = D.shard_total(N, k, G)
        sh = orc.OracleEnv(roms, n, 4, H.palette_rgb(), reset_cache_size=4, env_index_base=base)
        sh.reset(2)
        for t in range(steps):
            o, r, d = sh.step(acts[t, base:base + n])
            assert (o == ref[t][0][base:base + n]).all()
            assert (r == ref[t][1][base:base + n]).all() and (d == ref[t][2][base:base + n]).all()
        tot += sh.counters()
    assert (tot == full.counters()).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = torch.tensor([100 * (rank + 1), rank, -5 * rank, rank % 2], dtype=torch.int64)
        r = D.reduce_counters(c)
        m = D.max_over_ranks(1.5 + rank)
        base, n = D.shard(4096, rank)
        q.put((rank, r.tolist(), c.tolist(), m, base, n))
    finally:
        dist.destroy_process_group()


def test_gloo_counter_allreduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [sum(100 * (r + 1) for r in range(world)), sum(range(world)),
              sum(-5 * r for r in range(world)), sum(r % 2 for r in range(world))]
    for rank, reduced, local, m, base, n in res:
        assert reduced == expect                  # equals the host-side sum of per-rank counters
        assert local == [100 * (rank + 1), rank, -5 * rank, rank % 2]  # input untouched
        assert m == 1.5 + (world - 1)             # max over ranks
        assert (base, n) == (4096 * rank, 4096)


def test_oracle_pool_reproduces_one_process(orc):
    """tests/oracle_pool.py (the parallel oracle of the full-size GPU parity tests): chunks of
    global ids replayed in separate processes equal one sequential N-env oracle run, and a
    windowed replay from mid-run snapshots equals the continuation of that run."""
    import oracle_pool as OP
    roms = [games.build_rom("R1"), games.build_rom("R3")]
    N, T = 12, 16
    acts = H.random_actions(N, T, 8)
    full = orc.OracleEnv(roms, N, 4, H.palette_rgb(), reset_cache_size=3, max_episode_frames=20)
    full.reset(1)
    ref, st8 = [], None
    for t in range(T):
        if t == 8:
            st8 = full.get_state()
        ref.append(full.step(acts[t]))
    ids = np.array([0, 3, 4, 7, 11])
    cfg = dict(reset_cache_size=3, max_episode_frames=20)
    rew, done, dig, states, cnt = OP.trajectories(roms, ids, 4, acts, cfg=cfg, reset_seed=1, checkpoints={8})
    for t in range(T):
        assert (rew[t] == ref[t][1][ids]).all() and (done[t] == ref[t][2][ids]).all()
        assert (dig[t] == OP.digest_rows(ref[t][0][ids])).all()
    assert (states[8] == st8[ids]).all()
    steps, final = OP.windows(roms, ids, 4, st8[ids], acts[8:, ids], cfg=cfg, reset_seed=1)
    for k, (dg, r, d) in enumerate(steps):
        assert (dg == OP.digest_rows(ref[8 + k][0][ids])).all() and (r == ref[8 + k][1][ids]).all()
    assert (final == full.get_state()[ids]).all()
    assert done.sum() > 0
