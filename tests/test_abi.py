"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/cule.h declares
(no compute calls: this runs on the CPU-only build host)."""
import ctypes
import os
import re
import subprocess

import helpers as H

HEADER = os.path.join(H.ROOT, "include", "cule.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cule_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_1907_08467_b200 import _lib, build
    path = build.build()
    lib = ctypes.CDLL(path)
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_lib.EXPORTS) == names
    out = subprocess.run(["nm", "-D", path], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_sass_is_sm100a():
    from paper_1907_08467_b200 import build
    path = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls():
    # calls that touch no GPU: defaults, workspace sizing, argument validation
    from paper_1907_08467_b200 import _lib
    L = _lib.load()
    c = _lib.default_config()
    assert (c.obs_mode, c.reset_cache_size, c.startup_frames, c.max_random_frames, c.ystart,
            c.line_cap, c.score_addr, c.term_addr, c.term_mask) == (1, 30, 64, 30, 34, 1024, 0x80, 0x82, 1)
    n1 = L.cule_workspace_bytes(4096, 1, ctypes.byref(c))
    n2 = L.cule_workspace_bytes(8192, 1, ctypes.byref(c))
    assert n2 > n1 > 4096 * (256 + 33600)
    assert L.cule_workspace_bytes(0, 1, ctypes.byref(c)) == 0
    assert L.cule_workspace_bytes(16, 5, ctypes.byref(c)) == 0
    out = ctypes.c_void_p()
    rc = L.cule_create(None, None, 1, 16, 4, ctypes.byref(c), None, 0, ctypes.byref(out))
    assert rc == _lib.CULE_E_INVAL and b"null" in L.cule_last_error()
    assert L.cule_destroy(ctypes.c_void_p(12345)) == _lib.CULE_E_CLOSED


def test_env_rejects_bad_config_before_touching_the_gpu():
    # unknown config keys and obs modes are errors, not silently ignored
    import pytest
    from paper_1907_08467_b200 import Env
    from paper_1907_08467_b200.inputs import games
    rom = games.build_rom("R1")
    with pytest.raises(ValueError, match="obs_mode"):
        Env([rom], 4, 4, obs_mode="Gray84", device="cuda:0")
    with pytest.raises(ValueError, match="unknown config key 'idle_skp'"):
        Env([rom], 4, 4, device="cuda:0", idle_skp=1)
    with pytest.raises(ValueError, match="CUDA device only"):
        Env([rom], 4, 4, device="cpu")
