"""128-entry NTSC RGB palette (input data, shared by both sides as DATA only).

SPEC.md S:143 ("NTSC palette fixed as a 128-entry RGB table shipped as a data file") and
SURVEY.md §8(c).13 ledger row 15: Stella's table is not reproducible offline, so the table is
synthesized from a YIQ model (16 hues x 8 luminances) by `write_palette()` and committed as
`ntsc_palette.txt`.  Parity does not depend on the values (each side derives its own gray LUT
from the same RGB bytes, SURVEY.md §8(c).0 "Shared data only").

Palette index i = COLUxx >> 1 = (hue << 3) | lum.
"""
from __future__ import annotations

import math
import os

PALETTE_PATH = os.path.join(os.path.dirname(__file__), "ntsc_palette.txt")


def synthesize() -> list[tuple[int, int, int]]:
    out = []
    for hue in range(16):
        for lum in range(8):
            y = 0.06 + 0.88 * lum / 7.0 if (hue or lum) else 0.0
            if hue == 0:
                i_c = q_c = 0.0
            else:
                ang = math.radians(-33.0 + (hue - 1) * 24.0 + 180.0)
                sat = 0.18
                i_c, q_c = sat * math.cos(ang), sat * math.sin(ang)
            r = y + 0.956 * i_c + 0.621 * q_c
            g = y - 0.272 * i_c - 0.647 * q_c
            b = y - 1.106 * i_c + 1.703 * q_c
            out.append(tuple(max(0, min(255, int(round(c * 255)))) for c in (r, g, b)))
    return out


def write_palette(path: str = PALETTE_PATH) -> None:
    with open(path, "w") as f:
        f.write("# index R G B  (synthesized NTSC YIQ palette; see palette.py)\n")
        for i, (r, g, b) in enumerate(synthesize()):
            f.write(f"{i} {r} {g} {b}\n")


def load_palette(path: str = PALETTE_PATH) -> bytes:
    """Return 384 bytes: R,G,B for palette indices 0..127."""
    rgb = bytearray(384)
    seen = set()
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            i, r, g, b = (int(t) for t in line.split())
            rgb[3 * i:3 * i + 3] = bytes((r, g, b))
            seen.add(i)
    if seen != set(range(128)):
        raise ValueError("palette file must define indices 0..127")
    return bytes(rgb)


if __name__ == "__main__":
    write_palette()
