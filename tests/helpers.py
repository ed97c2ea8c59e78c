"""Test helpers: decode the documented 256-byte snapshot layout and common inputs.

Shared by the oracle tests and the GPU parity tests; holds none of the method's arithmetic.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1907_08467_b200.inputs import palette  # noqa: E402

# byte offsets of the snapshot
OFF = dict(A=0, X=1, Y=2, SP=3, P=4, bank=5, timer_v=16, timer_s=17, swcha=18, inpt4=19,
           vsync=24, vblank=25, nusiz0=26, nusiz1=27, colup0=28, colup1=29, colupf=30,
           colubk=31, ctrlpf=32, refp0=33, refp1=34, pf0=35, pf1=36, pf2=37, grp0new=38,
           grp0old=39, grp1new=40, grp1old=41, enam0=42, enam1=43, enablnew=44, enablold=45,
           hmp0=46, hmp1=47, hmm0=48, hmm1=49, hmbl=50, vdelp0=51, vdelp1=52, vdelbl=53,
           resmp0=54, resmp1=55, posP0=56, posP1=57, posM0=58, posM1=59, posBL=60,
           rom_id=61, fault=62)
RAM0 = 64
MACHINE_BYTES = list(range(0, 61)) + list(range(64, 192))


def u16(s, o):
    return int(s[o]) | (int(s[o + 1]) << 8)


def u32(s, o):
    return int(s[o]) | (int(s[o + 1]) << 8) | (int(s[o + 2]) << 16) | (int(s[o + 3]) << 24)


def i32(s, o):
    v = u32(s, o)
    return v - (1 << 32) if v & 0x80000000 else v


def pc(s):
    return u16(s, 6)


def fc(s):
    return u32(s, 8)


def timer_w(s):
    return i32(s, 12)


def coll(s):
    return u16(s, 20)


def comb_line(s):
    v = u16(s, 22)
    return v - 65536 if v & 0x8000 else v


def ram(s, addr):
    return int(s[RAM0 + (addr & 0x7F)])


def episode_frames(s):
    return u32(s, 192)


def episode_index(s):
    return u32(s, 196)


def episode_return(s):
    return i32(s, 200)


def prev_score(s):
    return u16(s, 204)


def set_pc(s, v):
    s[6] = v & 0xFF
    s[7] = (v >> 8) & 0xFF


def set_fc(s, v):
    for k in range(4):
        s[8 + k] = (v >> (8 * k)) & 0xFF


def palette_rgb() -> bytes:
    return palette.load_palette()


def gray_of_palette():
    """Gray LUT computed here from its definition (ITU-R 601 integer, half-up), §8(c).12."""
    rgb = np.frombuffer(palette_rgb(), np.uint8).reshape(128, 3).astype(np.int64)
    return ((299 * rgb[:, 0] + 587 * rgb[:, 1] + 114 * rgb[:, 2] + 500) // 1000).astype(np.uint8)


def random_actions(n_envs: int, n_steps: int, seed: int = 1234) -> np.ndarray:
    """i.i.d. uniform actions over the 18-action set (P:318-320 emulation-only random policy)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 18, size=(n_steps, n_envs), dtype=np.uint8)
