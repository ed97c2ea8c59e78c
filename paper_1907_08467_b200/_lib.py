"""ctypes binding of libcule (include/cule.h): argument marshalling only.

Every step of the emulation path runs in the CUDA kernels of libcule.so; this module only
passes pointers and sizes.  If the shared library is missing the import fails loudly — there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcule.so")

CULE_OK = 0
CULE_E_INVAL = -1
CULE_E_ROM_SIZE = -2
CULE_E_ROM_FAULT = -3
CULE_E_CUDA = -4
CULE_E_CLOSED = -5
CULE_OBS_RAW = 0
CULE_OBS_GRAY84 = 1
STATE_BYTES = 256

# every symbol include/cule.h declares
EXPORTS = ["cule_default_config", "cule_workspace_bytes", "cule_create", "cule_reset",
           "cule_step", "cule_step_host", "cule_get_state", "cule_set_state", "cule_counters",
           "cule_debug_exec", "cule_num_envs", "cule_frameskip", "cule_obs_bytes",
           "cule_engine", "cule_reset_stacked", "cule_step_stacked", "cule_vtrace", "cule_destroy", "cule_last_error",
           "cule_jit_prepare", "cule_jit_prepare_engine"]


class CuleConfig(ctypes.Structure):
    _fields_ = [("obs_mode", ctypes.c_int32), ("reset_cache_size", ctypes.c_int32),
                ("startup_frames", ctypes.c_int32), ("max_random_frames", ctypes.c_int32),
                ("max_episode_frames", ctypes.c_int32), ("line_cap", ctypes.c_int32),
                ("ystart", ctypes.c_int32), ("score_addr", ctypes.c_uint8),
                ("term_addr", ctypes.c_uint8), ("term_mask", ctypes.c_uint8),
                ("idle_skip", ctypes.c_uint8), ("seed", ctypes.c_uint64),
                ("env_index_base", ctypes.c_int64),
                ("palette_rgb", ctypes.POINTER(ctypes.c_uint8)),
                ("engine", ctypes.c_int32), ("tia_delays", ctypes.c_int32)]

CULE_ENGINE_AUTO, CULE_ENGINE_SIMT, CULE_ENGINE_SCALAR, CULE_ENGINE_JIT, CULE_ENGINE_VJIT = 0, 1, 2, 3, 4
CULE_ENGINE_WSVJIT = 5
ENGINE_NAMES = {CULE_ENGINE_SIMT: "simt", CULE_ENGINE_SCALAR: "scalar", CULE_ENGINE_JIT: "jit",
                CULE_ENGINE_VJIT: "vjit", CULE_ENGINE_WSVJIT: "wsvjit"}


class CuleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libcule error {code}: {msg}")
        self.code = code


_lib = None


def load():
    """Load libcule.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcule.so not built at {LIB_PATH}: run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    vp, u8p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint8)
    L.cule_default_config.argtypes = [ctypes.POINTER(CuleConfig)]
    L.cule_default_config.restype = None
    L.cule_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(CuleConfig)]
    L.cule_workspace_bytes.restype = ctypes.c_size_t
    L.cule_create.argtypes = [ctypes.POINTER(u8p), ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, ctypes.POINTER(CuleConfig), vp,
                              ctypes.c_size_t, ctypes.POINTER(vp)]
    L.cule_reset.argtypes = [vp, ctypes.c_uint64, vp, vp]
    L.cule_step.argtypes = [vp, vp, vp, vp, vp, vp]
    L.cule_step_host.argtypes = [vp, vp, vp, vp, vp, vp]
    L.cule_reset_stacked.argtypes = [vp, ctypes.c_uint64, vp, vp]
    f32 = ctypes.c_float
    L.cule_vtrace.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, f32, f32, f32, vp, vp, vp, vp]
    L.cule_step_stacked.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp, vp]
    L.cule_get_state.argtypes = [vp, vp, vp]
    L.cule_set_state.argtypes = [vp, vp, vp]
    L.cule_counters.argtypes = [vp, vp, vp]
    L.cule_debug_exec.argtypes = [vp, ctypes.c_int, vp, vp]
    L.cule_num_envs.argtypes = [vp]
    L.cule_frameskip.argtypes = [vp]
    L.cule_engine.argtypes = [vp]
    L.cule_obs_bytes.argtypes = [vp]
    L.cule_obs_bytes.restype = ctypes.c_size_t
    L.cule_destroy.argtypes = [vp]
    L.cule_jit_prepare.argtypes = [ctypes.POINTER(u8p), ctypes.POINTER(ctypes.c_size_t), ctypes.c_int, ctypes.c_int,
                                   ctypes.c_char_p, ctypes.c_size_t]
    L.cule_jit_prepare_engine.argtypes = [ctypes.POINTER(u8p), ctypes.POINTER(ctypes.c_size_t), ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]
    L.cule_last_error.argtypes = []
    L.cule_last_error.restype = ctypes.c_char_p
    for name in ("cule_create", "cule_reset", "cule_step", "cule_step_host", "cule_get_state",
                 "cule_reset_stacked", "cule_step_stacked", "cule_vtrace",
                 "cule_set_state", "cule_counters", "cule_debug_exec", "cule_num_envs",
                 "cule_frameskip", "cule_engine", "cule_destroy", "cule_jit_prepare", "cule_jit_prepare_engine"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> int:
    if rc < 0:
        raise CuleError(rc, load().cule_last_error().decode(errors="replace"))
    return rc


def default_config() -> CuleConfig:
    c = CuleConfig()
    load().cule_default_config(ctypes.byref(c))
    return c


def jit_prepare(roms, obs_mode: int = CULE_OBS_GRAY84, engine: int = CULE_ENGINE_JIT) -> str:
    """Translate + compile the step kernel of a translated engine (JIT or VJIT) for a ROM set
    into the on-disk cache (host only, no GPU needed; include/cule.h cule_jit_prepare_engine).
    Returns the library's summary line."""
    import numpy as np
    arrs = [np.frombuffer(bytes(r), np.uint8).copy() for r in roms]
    u8p = ctypes.POINTER(ctypes.c_uint8)
    ptrs = (u8p * len(arrs))(*[a.ctypes.data_as(u8p) for a in arrs])
    lens = (ctypes.c_size_t * len(arrs))(*[len(a) for a in arrs])
    buf = ctypes.create_string_buffer(512)
    check(load().cule_jit_prepare_engine(ptrs, lens, len(arrs), obs_mode, engine, buf, len(buf)))
    return buf.value.decode()
