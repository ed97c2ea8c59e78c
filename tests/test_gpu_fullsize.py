"""Full-size GPU parity at the bench's configurations (SURVEY.md §8(d) "Parity at scale";
VERDICT r01 "Next round" item 2).

  * cfg2 (4096 envs, R1, fs=4, GRAY84, the headline scalar engine): the full trajectory over a
    warm-up plus timed window of 310 steps for {g < 256} ∪ {g ≡ 0 mod 256} ∪ the first 256 envs
    that reset, compared every step (observation digest, reward, done) and at steps 100 / 300 /
    310 (the whole 256-byte state); windowed 10-step replays of ALL 4096 envs from their step-100
    and step-300 snapshots.
  * cfg4 (32768 envs, R1-R4 interleaved, the batched engine): the full trajectory of
    {g < 128} ∪ {g ≡ 0 mod 64} ∪ the first 128 resets, and windowed replays of every 8th env at
    steps 100 and 300.
  * Virtual shards: 8 sequential shards (env_index_base = k·N/8) of the cfg4 workload are byte-
    identical to one unsharded run, and at a size the oracle covers completely their summed
    counters equal the oracle's totals (SURVEY.md §8(e) pin).

The oracle runs in parallel host processes (tests/oracle_pool.py); the GPU is deterministic, so
the set of envs to check is chosen from one GPU pass and the outputs recorded in a second.
"""
import os

import numpy as np
import pytest

import helpers as H
import oracle_pool as OP
from paper_1907_08467_b200.inputs import games

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1907_08467_b200 import build
    build.build()
    import oracle
    oracle.build()


def gpu_run(roms, N, fs, acts, *, track=(), digest_all_steps=(), checkpoints=(), reset_seed=0, engine=None,
            engine_cfg=None, **cfg):
    """One GPU run through the C-ABI: rewards/dones of every env and step, digests of the
    tracked envs every step (of all envs on digest_all_steps), full snapshots before the
    checkpoint steps."""
    from paper_1907_08467_b200 import Env
    if engine_cfg is not None:
        cfg["engine"] = engine_cfg
    env = Env(roms, N, fs, **cfg)
    if engine is not None:
        assert env.engine == engine, (env.engine, engine)
    env.reset(reset_seed)
    T = len(acts)
    track = np.asarray(sorted(track), np.int64)
    tr_t = torch.from_numpy(track).to(env.device)
    rew = np.zeros((T, N), np.int32)
    done = np.zeros((T, N), np.uint8)
    dig, dig_all, states = {}, {}, {}
    d_acts = torch.from_numpy(acts).to(env.device)
    for t in range(T):
        if t in checkpoints:
            states[t] = env.get_state()
        o, r, d = env.step(d_acts[t])
        rew[t] = r.cpu().numpy()
        done[t] = d.cpu().numpy()
        if t in digest_all_steps:
            dig_all[t] = OP.digest_rows(o.cpu().numpy())
        if len(track):
            dig[t] = OP.digest_rows(o.index_select(0, tr_t).cpu().numpy())
    if T in checkpoints:
        states[T] = env.get_state()
    counters = env.counters().cpu().numpy()
    env.close()
    return dict(rew=rew, done=done, dig=dig, dig_all=dig_all, states=states, counters=counters, track=track)


def first_resets(done, k):
    """The first k envs to finish an episode (ordered by step, then env id)."""
    T, N = done.shape
    first = np.where(done.any(0), done.argmax(0), T)
    order = np.lexsort((np.arange(N), first))
    return order[first[order] < T][:k]


def check_full_size(roms, N, engine, base_set, n_resets, window_ids, T=310, window_steps=(100, 300), W=10):
    fs = 4
    acts = H.random_actions(N, T, 1234)
    # pass 1: which envs reset first (rewards/dones of every env are compared in pass 2 as well)
    p1 = gpu_run(roms, N, fs, acts, engine=engine, engine_cfg=engine)
    resets = first_resets(p1["done"], n_resets)
    assert len(resets) == n_resets, f"only {len(resets)} envs reset in {T} steps"
    track = np.union1d(base_set, resets)
    checkpoints = set(window_steps) | {s + W for s in window_steps} | {T}
    digest_all = {s + k for s in window_steps for k in range(W)}
    g = gpu_run(roms, N, fs, acts, track=track, digest_all_steps=digest_all, checkpoints=checkpoints,
                engine=engine, engine_cfg=engine)
    assert (g["rew"] == p1["rew"]).all() and (g["done"] == p1["done"]).all(), "GPU run not deterministic"

    # full trajectories of the tracked envs
    rew, done, dig, states, _ = OP.trajectories(roms, track, fs, acts, checkpoints=checkpoints)
    for t in range(T):
        assert (g["rew"][t, track] == rew[t]).all(), f"step {t}: rewards differ"
        assert (g["done"][t, track] == done[t]).all(), f"step {t}: dones differ"
        bad = np.nonzero(g["dig"][t] != dig[t])[0]
        assert len(bad) == 0, f"step {t}: observations differ for envs {track[bad][:8].tolist()}"
    for t in sorted(checkpoints):
        gs = g["states"][t][track]
        bad = np.nonzero((gs != states[t]).any(1))[0]
        assert len(bad) == 0, f"before step {t}: states differ for envs {track[bad][:8].tolist()}"
    n_done_tracked = int(done.sum())

    # windowed replays from the GPU's own snapshots
    for s in window_steps:
        ids = np.asarray(window_ids, np.int64)
        steps, final = OP.windows(roms, ids, fs, g["states"][s][ids], acts[s:s + W, ids])
        for k, (dg, r, d) in enumerate(steps):
            t = s + k
            assert (g["rew"][t, ids] == r).all() and (g["done"][t, ids] == d).all(), f"window {s}: step {t}"
            bad = np.nonzero(g["dig_all"][t][ids] != dg)[0]
            assert len(bad) == 0, f"window {s} step {t}: observations differ for envs {ids[bad][:8].tolist()}"
        bad = np.nonzero((g["states"][s + W][ids] != final).any(1))[0]
        assert len(bad) == 0, f"window {s}: final states differ for envs {ids[bad][:8].tolist()}"
    return len(track), n_done_tracked


@pytest.mark.parametrize("engine", ["jit", "scalar", "vjit"])
def test_cfg2_full_trajectory_and_windows(engine):
    N = 4096
    base = np.union1d(np.arange(256), np.arange(0, N, 256))
    n_track, n_done = check_full_size([games.build_rom("R1")], N, engine, base, 256, np.arange(N))
    assert n_track >= len(base) + 200 and n_done >= 256   # the resets overlap the base set a little


@pytest.mark.parametrize("engine", ["simt", "jit", "vjit", "wsvjit"])
def test_cfg4_full_trajectory_and_windows(engine):
    N = 32768
    roms = [games.build_rom(n) for n in ("R1", "R2", "R3", "R4")]
    base = np.union1d(np.arange(128), np.arange(0, N, 64))
    n_track, n_done = check_full_size(roms, N, engine, base, 128, np.arange(0, N, 8))
    assert n_track >= len(base) + 64 and n_done >= 128


def test_virtual_shards_byte_identical_at_cfg4():
    """8 shards of the cfg4 workload run one after another with env_index_base = k·N/8 reproduce
    the unsharded 32768-env run byte for byte (observations compared on the device, every step)."""
    from paper_1907_08467_b200 import Env
    from paper_1907_08467_b200 import dist as D
    roms = [games.build_rom(n) for n in ("R1", "R2", "R3", "R4")]
    N, G, T = 32768, 8, 30
    acts = torch.from_numpy(H.random_actions(N, T, 4321)).cuda()
    full = Env(roms, N, 4)
    full.reset(5)
    ref_obs, ref_rew, ref_done = [], [], []
    for t in range(T):
        o, r, d = full.step(acts[t])
        ref_obs.append(o.clone())
        ref_rew.append(r.clone())
        ref_done.append(d.clone())
    ref_state = full.get_state()
    ref_counters = full.counters().cpu().numpy()
    full.close()
    tot = np.zeros(4, np.int64)
    for k in range(G):
        base, n = D.shard_total(N, k, G)
        sh = Env(roms, n, 4, env_index_base=base)
        sh.reset(5)
        for t in range(T):
            o, r, d = sh.step(acts[t, base:base + n].contiguous())
            assert torch.equal(o, ref_obs[t][base:base + n]), (k, t)
            assert torch.equal(r, ref_rew[t][base:base + n]) and torch.equal(d, ref_done[t][base:base + n]), (k, t)
        assert (sh.get_state() == ref_state[base:base + n]).all(), k
        tot += sh.counters().cpu().numpy()
        sh.close()
    assert (tot == ref_counters).all(), (tot, ref_counters)


def test_sharded_counters_equal_oracle_totals():
    """At a size the oracle covers completely: Σ over 8 shards of the per-GPU counters
    {frames, episodes, return sum, faults} = the oracle's totals over all envs."""
    from paper_1907_08467_b200 import Env
    from paper_1907_08467_b200 import dist as D
    roms = [games.build_rom(n) for n in ("R1", "R2", "R3", "R4")]
    N, G, T = 2048, 8, 60
    acts = H.random_actions(N, T, 99)
    tot = np.zeros(4, np.int64)
    for k in range(G):
        base, n = D.shard_total(N, k, G)
        sh = Env(roms, n, 4, env_index_base=base)
        sh.reset(0)
        d_acts = torch.from_numpy(acts[:, base:base + n].copy()).cuda()
        for t in range(T):
            sh.step(d_acts[t])
        tot += sh.counters().cpu().numpy()
        sh.close()
    _, done, _, _, counters = OP.trajectories(roms, np.arange(N), 4, acts, digest_steps=set())
    assert (tot == counters).all(), (tot, counters)
    assert tot[0] == N * 4 * T and tot[1] == int(done.sum()) > 0
