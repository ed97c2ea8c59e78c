"""paper_1907_08467_b200 — B200-native batched Atari 2600 emulation (the CuLE hot path).

    from paper_1907_08467_b200 import Env
    env = Env([rom_bytes], num_envs=4096, frameskip=4)      # GRAY84 observations
    obs = env.reset(seed=0)
    obs, rewards, dones = env.step(actions_u8_cuda)

The work happens in libcule.so (csrc/, sm_100a); see DESIGN.md.
"""
from .env import Env  # noqa: F401

__all__ = ["Env"]
