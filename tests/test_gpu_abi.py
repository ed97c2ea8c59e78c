"""Boundary behaviour on the GPU: snapshot validation, host-buffer checks, error codes
(include/cule.h)."""
import numpy as np
import pytest
import torch

from paper_1907_08467_b200 import Env, _lib
from paper_1907_08467_b200.inputs import games

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    rom = games.build_rom("R1")
    e = Env([rom, games.build_rom("R2")], 8, 4, reset_cache_size=2)
    e.reset(0)
    yield e
    e.close()


@pytest.mark.parametrize("off,val,msg", [(61, 2, "rom_id"), (5, 2, "bank"), (17, 4, "timer shift"),
                                         (56, 160, "position"), (60, 255, "position"), (62, 3, "fault"),
                                         (11, 0x10, "line cap")])
def test_set_state_rejects_out_of_model_snapshots(env, off, val, msg):
    good = env.get_state()
    bad = good.copy()
    bad[5, off] = val
    with pytest.raises(_lib.CuleError) as ei:
        env.set_state(bad)
    assert ei.value.code == _lib.CULE_E_INVAL and msg in str(ei.value)
    assert (env.get_state() == good).all()      # nothing was uploaded
    env.set_state(good)                          # a valid snapshot still loads


def test_set_state_bank_of_f8_rom(env):
    s = env.get_state()
    s[1, 5] = 1          # env 1 runs R2 (F8, 2 banks): bank 1 is valid
    env.set_state(s)
    s[0, 5] = 1          # env 0 runs R1 (4K): bank 1 is not
    with pytest.raises(_lib.CuleError):
        env.set_state(s)


def test_step_host_checks_buffers(env):
    n = env.num_envs
    a = torch.zeros(n, dtype=torch.uint8)
    obs = torch.zeros(n, 84, 84, dtype=torch.uint8)
    rew = torch.zeros(n, dtype=torch.int32)
    done = torch.zeros(n, dtype=torch.uint8)
    env.step_host(a, obs, rew, done)
    env.step_host(a, None, rew, done)
    with pytest.raises(ValueError, match="h_obs"):
        env.step_host(a, torch.zeros(n - 1, 84, 84, dtype=torch.uint8), rew, done)
    with pytest.raises(ValueError, match="h_rewards"):
        env.step_host(a, obs, torch.zeros(n, dtype=torch.int64), done)
    with pytest.raises(ValueError, match="h_actions"):
        env.step_host(a.cuda(), obs, rew, done)


def test_handle_runs_on_its_own_device_stream(env):
    # the env's calls take the current stream of the env's device; an explicit stream works too
    s = torch.cuda.Stream(device=env.device)
    a = torch.zeros(env.num_envs, dtype=torch.uint8, device=env.device)
    with torch.cuda.stream(s):
        env.step(a, stream=s)
    s.synchronize()
    assert np.isfinite(env.rewards.cpu().numpy()).all()


def test_vtrace_checks_out_buffers():
    from paper_1907_08467_b200 import vtrace
    T, B = 4, 8
    f = lambda: torch.zeros(T, B, device="cuda")  # noqa: E731
    args = (f(), f(), torch.zeros(B, device="cuda"), f(), f(), torch.zeros(T, B, dtype=torch.uint8, device="cuda"))
    vtrace.vtrace(*args, gamma=0.99)
    with pytest.raises(ValueError, match="out"):
        vtrace.vtrace(*args, gamma=0.99, out=(f(), f(), torch.zeros(T, B + 1, device="cuda")))
    with pytest.raises(ValueError, match="out"):
        vtrace.vtrace(*args, gamma=0.99, out=(f(), f(), torch.zeros(T, B, dtype=torch.float64, device="cuda")))
