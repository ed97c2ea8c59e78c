"""`Env`: the Python face of libcule — batched Atari 2600 environments on one GPU.

PyTorch supplies device memory (workspace, observation/reward/done buffers) and streams; the
library does all of the work on the device ("CuLE comes with a python
interface"; SPEC.md S:541-566 flat create/step/reset/close, preallocated reusable buffers).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .inputs import palette as _palette


def _stream_ptr(stream=None, device=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


class Env:
    """N environments; env with global id g = env_index_base + i runs roms[g % len(roms)].

    obs_mode: 'gray84' -> obs u8[N, 84, 84]; 'raw' -> obs u8[N, 210, 160] palette indices.
    Output tensors are preallocated once and overwritten by every step.
    """

    def __init__(self, roms, num_envs: int, frameskip: int = 4, obs_mode: str = "gray84",
                 seed: int = 0, device=None, env_index_base: int = 0, **cfg):
        L = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("Env runs on a CUDA device only (no CPU fallback)")
        roms = [bytes(r) for r in roms]
        self.num_envs = int(num_envs)
        self.frameskip = int(frameskip)
        if obs_mode not in ("gray84", "raw"):
            raise ValueError(f"obs_mode must be 'gray84' or 'raw', got {obs_mode!r}")
        c = _lib.default_config()
        c.obs_mode = _lib.CULE_OBS_GRAY84 if obs_mode == "gray84" else _lib.CULE_OBS_RAW
        c.seed = seed
        c.env_index_base = env_index_base
        fields = {f for f, _ in _lib.CuleConfig._fields_} - {"obs_mode", "palette_rgb"}
        if isinstance(cfg.get("engine"), str):
            names = {v: k for k, v in _lib.ENGINE_NAMES.items()} | {"auto": _lib.CULE_ENGINE_AUTO}
            if cfg["engine"] not in names:
                raise ValueError(f"engine must be one of {sorted(names)}")
            cfg["engine"] = names[cfg["engine"]]
        for k, v in cfg.items():
            if k not in fields:
                raise ValueError(f"unknown config key {k!r}; valid keys: {sorted(fields)}")
            setattr(c, k, v)
        self._pal = np.frombuffer(_palette.load_palette(), np.uint8).copy()
        c.palette_rgb = self._pal.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        self.cfg = c
        self.obs_mode = obs_mode
        with torch.cuda.device(self.device):
            nbytes = L.cule_workspace_bytes(self.num_envs, len(roms), ctypes.byref(c))
            if nbytes == 0:
                raise _lib.CuleError(_lib.CULE_E_INVAL, "bad workspace request")
            self._ws_raw = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
            base = self._ws_raw.data_ptr()
            off = (-base) % 256
            self._ws_ptr = base + off
            self._roms = [np.frombuffer(r, np.uint8).copy() for r in roms]
            arr = (ctypes.POINTER(ctypes.c_uint8) * len(roms))(
                *[r.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)) for r in self._roms])
            lens = (ctypes.c_size_t * len(roms))(*[len(r) for r in roms])
            h = ctypes.c_void_p()
            _lib.check(L.cule_create(arr, lens, len(roms), self.num_envs, self.frameskip,
                                     ctypes.byref(c), ctypes.c_void_p(self._ws_ptr), nbytes,
                                     ctypes.byref(h)))
            self._h = h
            shape = (84, 84) if obs_mode == "gray84" else (210, 160)
            self.obs = torch.zeros((self.num_envs,) + shape, dtype=torch.uint8, device=self.device)
            self.rewards = torch.zeros(self.num_envs, dtype=torch.int32, device=self.device)
            self.dones = torch.zeros(self.num_envs, dtype=torch.uint8, device=self.device)
            self._counters = torch.zeros(4, dtype=torch.int64, device=self.device)
        self.obs_bytes = int(np.prod(shape))
        self.engine = _lib.ENGINE_NAMES[_lib.check(L.cule_engine(self._h))]

    def _sp(self, stream) -> int:
        """The caller's stream, else the current stream of the env's device (not of whatever
        device happens to be current); the library switches to the env's device itself."""
        if stream is not None and stream.device != self.device:
            raise ValueError("stream must belong to the env's device")
        return _stream_ptr(stream, self.device)

    # -- core calls ----------------------------------------------------------------------------
    def reset(self, seed: int = 0, stream=None) -> torch.Tensor:
        _lib.check(_lib.load().cule_reset(self._h, seed, ctypes.c_void_p(self.obs.data_ptr()),
                                          ctypes.c_void_p(self._sp(stream))))
        return self.obs

    def step(self, actions: torch.Tensor, stream=None):
        if actions.dtype != torch.uint8 or actions.device != self.device or actions.numel() != self.num_envs:
            raise ValueError("actions must be a uint8 tensor of N elements on the env's device")
        actions = actions.contiguous()
        _lib.check(_lib.load().cule_step(self._h, ctypes.c_void_p(actions.data_ptr()),
                                         ctypes.c_void_p(self.obs.data_ptr()),
                                         ctypes.c_void_p(self.rewards.data_ptr()),
                                         ctypes.c_void_p(self.dones.data_ptr()),
                                         ctypes.c_void_p(self._sp(stream))))
        return self.obs, self.rewards, self.dones

    # -- inference path: frame stack (R#32) ------------------
    def new_stack(self) -> torch.Tensor:
        """A device frame stack u8[N, 4, 84, 84] for reset_stacked / step_stacked."""
        if self.obs_mode != "gray84":
            raise ValueError("frame stacks need gray84 observations")
        return torch.zeros((self.num_envs, 4, 84, 84), dtype=torch.uint8, device=self.device)

    def reset_stacked(self, stack: torch.Tensor, seed: int = 0, stream=None) -> torch.Tensor:
        self._check_stack(stack)
        _lib.check(_lib.load().cule_reset_stacked(self._h, seed, ctypes.c_void_p(stack.data_ptr()),
                                                  ctypes.c_void_p(self._sp(stream))))
        return stack

    def step_stacked(self, actions: torch.Tensor, stack: torch.Tensor, slot: int, stream=None):
        """One step writing each env's observation into stack[:, slot] (slot rotates 0..3); an env
        that ended its episode gets its new start observation in all four slots."""
        self._check_stack(stack)
        if actions.dtype != torch.uint8 or actions.device != self.device or actions.numel() != self.num_envs:
            raise ValueError("actions must be a uint8 tensor of N elements on the env's device")
        actions = actions.contiguous()
        _lib.check(_lib.load().cule_step_stacked(self._h, ctypes.c_void_p(actions.data_ptr()),
                                                 ctypes.c_void_p(stack.data_ptr()), int(slot),
                                                 ctypes.c_void_p(self.rewards.data_ptr()),
                                                 ctypes.c_void_p(self.dones.data_ptr()),
                                                 ctypes.c_void_p(self._sp(stream))))
        return self.rewards, self.dones

    def _check_stack(self, stack: torch.Tensor) -> None:
        if (stack.dtype != torch.uint8 or stack.device != self.device or not stack.is_contiguous()
                or tuple(stack.shape) != (self.num_envs, 4, 84, 84)):
            raise ValueError("stack must be a contiguous uint8 tensor [N, 4, 84, 84] on the env's device")

    def step_host(self, h_actions: torch.Tensor, h_obs, h_rewards: torch.Tensor,
                  h_dones: torch.Tensor, stream=None):
        """Host-buffer step (pinned CPU tensors): copies in, steps, copies out, synchronises.
        h_actions u8[N], h_obs u8[N, *obs_shape] or None, h_rewards i32[N], h_dones u8[N]: all
        contiguous CPU tensors (pinned recommended); the library writes exactly these sizes."""
        n = self.num_envs
        for name, t, dt, numel in (("h_actions", h_actions, torch.uint8, n),
                                   ("h_obs", h_obs, torch.uint8, n * self.obs_bytes),
                                   ("h_rewards", h_rewards, torch.int32, n), ("h_dones", h_dones, torch.uint8, n)):
            if t is None and name == "h_obs":
                continue
            if (not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != dt
                    or not t.is_contiguous() or t.numel() != numel):
                raise ValueError(f"{name} must be a contiguous CPU {dt} tensor of {numel} elements")
        _lib.check(_lib.load().cule_step_host(
            self._h, ctypes.c_void_p(h_actions.data_ptr()),
            ctypes.c_void_p(h_obs.data_ptr() if h_obs is not None else 0),
            ctypes.c_void_p(h_rewards.data_ptr()), ctypes.c_void_p(h_dones.data_ptr()),
            ctypes.c_void_p(self._sp(stream))))

    def get_state(self, stream=None) -> np.ndarray:
        out = np.zeros((self.num_envs, _lib.STATE_BYTES), np.uint8)
        _lib.check(_lib.load().cule_get_state(self._h, ctypes.c_void_p(out.ctypes.data),
                                              ctypes.c_void_p(self._sp(stream))))
        return out

    def set_state(self, states: np.ndarray, stream=None) -> None:
        s = np.ascontiguousarray(states, dtype=np.uint8)
        if s.shape != (self.num_envs, _lib.STATE_BYTES):
            raise ValueError("states must be u8[N, 256]")
        _lib.check(_lib.load().cule_set_state(self._h, ctypes.c_void_p(s.ctypes.data),
                                              ctypes.c_void_p(self._sp(stream))))

    def counters(self, stream=None) -> torch.Tensor:
        """int64[4] on the device: frames, episodes finished, sum of episode returns, faults."""
        _lib.check(_lib.load().cule_counters(self._h, ctypes.c_void_p(self._counters.data_ptr()),
                                             ctypes.c_void_p(self._sp(stream))))
        return self._counters

    def counters_into(self, out: torch.Tensor, stream=None) -> torch.Tensor:
        """Like counters(), into a caller-owned int64[4] device tensor (stream-ordered copy)."""
        if out.dtype != torch.int64 or out.device != self.device or out.numel() != 4 or not out.is_contiguous():
            raise ValueError("out must be a contiguous int64[4] tensor on the env's device")
        _lib.check(_lib.load().cule_counters(self._h, ctypes.c_void_p(out.data_ptr()),
                                             ctypes.c_void_p(self._sp(stream))))
        return out

    def debug_exec(self, n_instr: int, stream=None) -> torch.Tensor:
        status = torch.zeros(self.num_envs, dtype=torch.int32, device=self.device)
        _lib.check(_lib.load().cule_debug_exec(self._h, n_instr, ctypes.c_void_p(status.data_ptr()),
                                               ctypes.c_void_p(self._sp(stream))))
        return status

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            torch.cuda.synchronize(self.device)
            _lib.check(_lib.load().cule_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
