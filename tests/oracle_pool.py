"""Run the CPU oracle over many environments in parallel host processes (SURVEY.md §8(d) "the
oracle runs in P host processes").

Test infrastructure: workers import only numpy and the oracle.  Envs are independent and keyed by
their global id (R#22), so a chunk of global ids replayed in its own process with
`OracleEnv.set_env_ids` reproduces those envs of an N-env run exactly.

Observations are compared through an 8-byte BLAKE2b digest per (step, env); the GPU side uses the
same `digest_rows` on the bytes it copies back.
"""
from __future__ import annotations

import hashlib
import multiprocessing as mp
import os

import numpy as np


def digest_rows(obs: np.ndarray) -> np.ndarray:
    """u64 digest of every row of obs[n, ...] (BLAKE2b, 8 bytes)."""
    flat = np.ascontiguousarray(obs).reshape(len(obs), -1)
    out = np.empty(len(flat), np.uint64)
    for i in range(len(flat)):
        out[i] = int.from_bytes(hashlib.blake2b(flat[i].tobytes(), digest_size=8).digest(), "little")
    return out


def _palette():
    from paper_1907_08467_b200.inputs import palette
    return palette.load_palette()


def _trajectory_worker(args):
    roms, ids, fs, obs_mode, cfg, acts, reset_seed, checkpoints, digest_steps = args
    import oracle
    env = oracle.OracleEnv(roms, len(ids), fs, _palette(), obs_mode=obs_mode, **cfg)
    env.set_env_ids(ids)
    env.reset(reset_seed)
    T = len(acts)
    rew = np.zeros((T, len(ids)), np.int32)
    done = np.zeros((T, len(ids)), np.uint8)
    dig = {}
    states = {}
    for t in range(T):
        if t in checkpoints:
            states[t] = env.get_state()
        o, r, d = env.step(acts[t])
        rew[t], done[t] = r, d
        if digest_steps is None or t in digest_steps:
            dig[t] = digest_rows(o)
    if T in checkpoints:
        states[T] = env.get_state()
    return rew, done, dig, states, env.counters()


def _window_worker(args):
    roms, ids, fs, obs_mode, cfg, states, acts, reset_seed = args
    import oracle
    env = oracle.OracleEnv(roms, len(ids), fs, _palette(), obs_mode=obs_mode, **cfg)
    env.set_env_ids(ids)
    env.reset(reset_seed)          # pick seed of the run the snapshots come from
    env.set_state(states)
    out = []
    for t in range(len(acts)):
        o, r, d = env.step(acts[t])
        out.append((digest_rows(o), r.copy(), d.copy()))
    return out, env.get_state()


def _pool(n_tasks):
    procs = max(1, min(n_tasks, len(os.sched_getaffinity(0))))
    return mp.get_context("spawn").Pool(procs)


def _chunks(ids, n):
    ids = np.asarray(ids, np.int64)
    k = max(1, min(len(ids), n))
    return [c for c in np.array_split(ids, k) if len(c)]


def trajectories(roms, ids, fs, acts_all, *, obs_mode=1, cfg=None, reset_seed=0, checkpoints=(),
                 digest_steps=None):
    """Replay global env ids `ids` from reset(reset_seed) through acts_all[T, N].  Returns
    (rewards [T, n], dones [T, n], {t: digests [n]}, {t: states [n, 256]} taken before step t,
    summed counters int64[4]) in the order of `ids`."""
    cfg = dict(cfg or {})
    ids = np.asarray(ids, np.int64)
    chunks = _chunks(ids, 4 * len(os.sched_getaffinity(0)))
    tasks = [(roms, c, fs, obs_mode, cfg, np.ascontiguousarray(acts_all[:, c]), reset_seed,
              set(checkpoints), None if digest_steps is None else set(digest_steps)) for c in chunks]
    with _pool(len(tasks)) as p:
        res = p.map(_trajectory_worker, tasks)
    rew = np.concatenate([r[0] for r in res], 1)
    done = np.concatenate([r[1] for r in res], 1)
    steps = res[0][2].keys()
    dig = {t: np.concatenate([r[2][t] for r in res]) for t in steps}
    states = {t: np.concatenate([r[3][t] for r in res]) for t in res[0][3]}
    counters = np.sum([r[4] for r in res], 0)
    return rew, done, dig, states, counters


def windows(roms, ids, fs, states, acts, *, obs_mode=1, cfg=None, reset_seed=0):
    """Load snapshots states[n, 256] of global ids `ids` and replay acts[W, n].  Returns
    ([(digests [n], rewards [n], dones [n]) per step], final states [n, 256])."""
    cfg = dict(cfg or {})
    ids = np.asarray(ids, np.int64)
    pos = np.arange(len(ids))
    chunks = _chunks(pos, 4 * len(os.sched_getaffinity(0)))
    tasks = [(roms, ids[c], fs, obs_mode, cfg, np.ascontiguousarray(states[c]),
              np.ascontiguousarray(acts[:, c]), reset_seed) for c in chunks]
    with _pool(len(tasks)) as p:
        res = p.map(_window_worker, tasks)
    W = len(acts)
    steps = [(np.concatenate([r[0][t][0] for r in res]), np.concatenate([r[0][t][1] for r in res]),
              np.concatenate([r[0][t][2] for r in res])) for t in range(W)]
    return steps, np.concatenate([r[1] for r in res])
