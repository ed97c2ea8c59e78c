"""ctypes loader for the CPU oracle (liboracle.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SOURCES = [os.path.join(HERE, "cule_oracle.c")]
HEADERS = [os.path.join(HERE, "oracle.h")]

FB_W, FB_H = 160, 210
STATE_BYTES = 256


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, -O2, no vectorisation flags beyond -O2)."""
    newest = max(os.path.getmtime(p) for p in SOURCES + HEADERS)
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= newest:
        return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Wno-unused-parameter",
                           "-shared", "-fPIC", "-o", tmp] + SOURCES)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class OrcConfig(ctypes.Structure):
    _fields_ = [("obs_mode", ctypes.c_int32), ("reset_cache_size", ctypes.c_int32),
                ("startup_frames", ctypes.c_int32), ("max_random_frames", ctypes.c_int32),
                ("max_episode_frames", ctypes.c_int32), ("line_cap", ctypes.c_int32),
                ("ystart", ctypes.c_int32), ("score_addr", ctypes.c_uint8),
                ("term_addr", ctypes.c_uint8), ("term_mask", ctypes.c_uint8),
                ("tia_delays", ctypes.c_uint8), ("seed", ctypes.c_uint64),
                ("env_index_base", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.orc_power_on.argtypes = [u8p, ctypes.c_size_t, u8p]
        L.orc_exec.argtypes = [u8p, ctypes.c_size_t, u8p, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_int64)]
        L.orc_run_frame.argtypes = [u8p, ctypes.c_size_t, u8p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, u8p, ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64)]
        L.orc_run_frame_ex.argtypes = [u8p, ctypes.c_size_t, u8p, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, u8p, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.orc_gray_lut.argtypes = [u8p, u8p]
        L.orc_area84.argtypes = [u8p, u8p]
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_hash2.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.orc_hash2.restype = ctypes.c_uint64
        L.orc_default_config.argtypes = [ctypes.POINTER(OrcConfig)]
        L.orc_create.argtypes = [ctypes.POINTER(u8p), ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, ctypes.POINTER(OrcConfig), u8p,
                                 ctypes.POINTER(ctypes.c_int)]
        L.orc_create.restype = ctypes.c_void_p
        L.orc_set_env_ids.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
        L.orc_reset.argtypes = [ctypes.c_void_p, ctypes.c_uint64, u8p]
        L.orc_step.argtypes = [ctypes.c_void_p, u8p, u8p, ctypes.POINTER(ctypes.c_int32), u8p]
        L.orc_reset_stacked.argtypes = [ctypes.c_void_p, ctypes.c_uint64, u8p]
        L.orc_step_stacked.argtypes = [ctypes.c_void_p, u8p, u8p, ctypes.c_int, ctypes.POINTER(ctypes.c_int32), u8p]
        L.orc_get_state.argtypes = [ctypes.c_void_p, u8p]
        L.orc_set_state.argtypes = [ctypes.c_void_p, u8p]
        L.orc_counters.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
        L.orc_get_cache.argtypes = [ctypes.c_void_p, u8p, u8p]
        L.orc_destroy.argtypes = [ctypes.c_void_p]
    return _lib


def _u8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _rom_arr(rom: bytes) -> np.ndarray:
    return np.frombuffer(bytes(rom), dtype=np.uint8).copy()


def power_on(rom: bytes) -> np.ndarray:
    s = np.zeros(STATE_BYTES, np.uint8)
    r = _rom_arr(rom)
    if lib().orc_power_on(_u8(r), len(r), _u8(s)) != 0:
        raise ValueError("bad ROM size")
    return s


def exec_instr(rom: bytes, state: np.ndarray, n: int = 1, line_cap: int = 1024):
    """Execute n instructions in place; returns (status, cycles)."""
    r = _rom_arr(rom)
    cyc = ctypes.c_int64(0)
    st = lib().orc_exec(_u8(r), len(r), _u8(state), n, line_cap, ctypes.byref(cyc))
    return st, cyc.value


def run_frame(rom: bytes, state: np.ndarray, action: int = -1, ystart: int = 34,
              line_cap: int = 1024, render: bool = True, tia_delays: int = 0):
    """Run one frame in place; returns (status, fb or None, instructions, scanlines).
    tia_delays=1: the delayed register effects of DESIGN.md R#35."""
    r = _rom_arr(rom)
    fb = np.zeros(FB_W * FB_H, np.uint8) if render else None
    ic = ctypes.c_int64(0)
    lines = ctypes.c_int64(0)
    st = lib().orc_run_frame_ex(_u8(r), len(r), _u8(state), action, ystart, line_cap,
                                _u8(fb) if render else None, ctypes.byref(ic), ctypes.byref(lines),
                                int(tia_delays))
    return st, (fb.reshape(FB_H, FB_W) if render else None), ic.value, lines.value


def gray_lut(rgb: bytes) -> np.ndarray:
    src = np.frombuffer(rgb, np.uint8).copy()
    out = np.zeros(128, np.uint8)
    lib().orc_gray_lut(_u8(src), _u8(out))
    return out


def area84(gray: np.ndarray) -> np.ndarray:
    g = np.ascontiguousarray(gray, dtype=np.uint8).reshape(-1)
    assert g.size == FB_W * FB_H
    out = np.zeros(84 * 84, np.uint8)
    lib().orc_area84(_u8(g), _u8(out))
    return out.reshape(84, 84)


def default_config(**kw) -> OrcConfig:
    c = OrcConfig()
    lib().orc_default_config(ctypes.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class OracleEnv:
    """Sequential CPU oracle over N envs (mirror of the cule_* env calls)."""

    def __init__(self, roms, num_envs: int, frameskip: int, palette_rgb: bytes, **cfg):
        L = lib()
        self.cfg = default_config(**cfg)
        self.num_envs = num_envs
        self.frameskip = frameskip
        self._roms = [_rom_arr(r) for r in roms]
        arr = (ctypes.POINTER(ctypes.c_uint8) * len(roms))(*[_u8(r) for r in self._roms])
        lens = (ctypes.c_size_t * len(roms))(*[len(r) for r in self._roms])
        pal = np.frombuffer(palette_rgb, np.uint8).copy()
        err = ctypes.c_int(0)
        self.h = L.orc_create(arr, lens, len(roms), num_envs, frameskip, ctypes.byref(self.cfg),
                              _u8(pal), ctypes.byref(err))
        if not self.h:
            raise ValueError(f"orc_create failed: {err.value}")
        self.obs_shape = (FB_H, FB_W) if self.cfg.obs_mode == 0 else (84, 84)

    def set_env_ids(self, gids):
        g = np.ascontiguousarray(gids, dtype=np.int64)
        assert g.size == self.num_envs
        lib().orc_set_env_ids(self.h, g.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))

    def reset(self, seed: int = 0) -> np.ndarray:
        obs = np.zeros((self.num_envs,) + self.obs_shape, np.uint8)
        lib().orc_reset(self.h, seed, _u8(obs))
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.uint8)
        obs = np.zeros((self.num_envs,) + self.obs_shape, np.uint8)
        rew = np.zeros(self.num_envs, np.int32)
        done = np.zeros(self.num_envs, np.uint8)
        lib().orc_step(self.h, _u8(a), _u8(obs), rew.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                       _u8(done))
        return obs, rew, done

    # frame stack of the inference path (GRAY84; R#32)
    def reset_stacked(self, seed: int = 0) -> np.ndarray:
        stack = np.zeros((self.num_envs, 4) + self.obs_shape, np.uint8)
        lib().orc_reset_stacked(self.h, seed, _u8(stack))
        return stack

    def step_stacked(self, actions, stack: np.ndarray, slot: int):
        """One step; `stack` (u8[N][4][84][84]) is updated in place."""
        assert stack.flags.c_contiguous and stack.shape == (self.num_envs, 4) + self.obs_shape
        a = np.ascontiguousarray(actions, dtype=np.uint8)
        rew = np.zeros(self.num_envs, np.int32)
        done = np.zeros(self.num_envs, np.uint8)
        rc = lib().orc_step_stacked(self.h, _u8(a), _u8(stack), slot,
                                    rew.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _u8(done))
        assert rc == 0
        return rew, done

    def get_state(self) -> np.ndarray:
        s = np.zeros((self.num_envs, STATE_BYTES), np.uint8)
        lib().orc_get_state(self.h, _u8(s))
        return s

    def set_state(self, s: np.ndarray) -> None:
        s = np.ascontiguousarray(s, dtype=np.uint8)
        lib().orc_set_state(self.h, _u8(s))

    def counters(self) -> np.ndarray:
        c = np.zeros(4, np.int64)
        lib().orc_counters(self.h, c.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        return c

    def cache(self):
        n = len(self._roms) * self.cfg.reset_cache_size
        st = np.zeros((n, STATE_BYTES), np.uint8)
        ob = np.zeros((n,) + self.obs_shape, np.uint8)
        lib().orc_get_cache(self.h, _u8(st), _u8(ob))
        return st, ob

    def close(self):
        if self.h:
            lib().orc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
