"""Pins for the oracle's frame stack of the inference path (DESIGN.md
R#32): checked against the oracle's plain step outputs and its reset cache, not by restating
the rule.  The entry an env was reset to is identified by content (its machine part equals
exactly one cache entry's), not by re-deriving the pick."""
import numpy as np

import helpers as H
from paper_1907_08467_b200.inputs import games

R1 = games.build_rom("R1")
MACHINE = np.r_[0:61, 64:192]  # snapshot bytes a reset copies from the cache entry


def make(orc, n=6, **cfg):
    cfg.setdefault("reset_cache_size", 5)
    return orc.OracleEnv([R1], n, 4, H.palette_rgb(), obs_mode=1, **cfg)


def test_reset_stacked_fills_every_slot_with_the_reset_observation(orc):
    plain, stacked = make(orc), make(orc)
    obs = plain.reset(7)
    stack = stacked.reset_stacked(7)
    assert stack.shape == (6, 4, 84, 84)
    for k in range(4):
        assert (stack[:, k] == obs).all()
    assert (plain.get_state() == stacked.get_state()).all()


def test_ring_order_and_episode_starts(orc):
    # an episode cap of 12 frames (3 steps at fs=4) forces episode ends on every env
    plain, stacked = make(orc, max_episode_frames=12), make(orc, max_episode_frames=12)
    plain.reset(3)
    stack = stacked.reset_stacked(3)
    cache_states, cache_obs = plain.cache()
    history = [[] for _ in range(6)]  # observations of each env's current episode, in order
    rng = np.random.default_rng(5)
    n_done = 0
    for t in range(11):
        a = rng.integers(0, 18, 6, dtype=np.uint8)
        before = stack.copy()
        o, r, d = plain.step(a)
        r2, d2 = stacked.step_stacked(a, stack, t % 4)
        assert (r == r2).all() and (d == d2).all()
        states = plain.get_state()
        assert (states == stacked.get_state()).all()
        for i in range(6):
            if d[i]:
                n_done += 1
                match = np.nonzero((cache_states[:, MACHINE] == states[i, MACHINE]).all(1))[0]
                assert len(match) == 1
                for k in range(4):
                    assert (stack[i, k] == cache_obs[match[0]]).all()
                history[i] = [cache_obs[match[0]]]
            else:
                assert (stack[i, t % 4] == o[i]).all()
                for k in range(4):
                    if k != t % 4:
                        assert (stack[i, k] == before[i, k]).all()
                history[i].append(o[i])
                # slots slot+1 .. slot (mod 4) run oldest -> newest over the episode so far
                seq = [stack[i, (t % 4 + 1 + k) % 4] for k in range(4)]
                for k in range(min(4, len(history[i]))):
                    assert (seq[3 - k] == history[i][-1 - k]).all()
    assert n_done >= 12


def test_bad_slot_rejected(orc):
    e = make(orc, n=2)
    stack = e.reset_stacked(0)
    import pytest
    with pytest.raises(AssertionError):
        e.step_stacked(np.zeros(2, np.uint8), stack, 4)
