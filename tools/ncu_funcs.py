"""Aggregate the per-line ncu source counters of a .ncu-rep by function (line ranges found by
scanning the source file for top-level function/struct-method heads).

    python tools/ncu_funcs.py gpurun_out/prof.ncu-rep paper_1907_08467_b200/csrc/scalar_tia.cuh
"""
import re
import subprocess
import sys


def ranges(path):
    heads = []
    for i, line in enumerate(open(path), 1):
        m = re.match(r"\s*(?:__device__|template).*?\b([A-Za-z_][A-Za-z0-9_]*)\s*\(", line)
        if m and ("__device__" in line):
            heads.append((i, m.group(1)))
    out = []
    for j, (i, name) in enumerate(heads):
        end = heads[j + 1][0] - 1 if j + 1 < len(heads) else 10 ** 9
        out.append((i, end, name))
    return out


def main(rep, src):
    fname = src.split("/")[-1]
    rs = ranges(src)
    txt = subprocess.run([sys.executable, "tools/ncu_source.py", rep, "100000"], capture_output=True, text=True).stdout
    acc = {}
    for line in txt.splitlines():
        m = re.match(r"\s*([\d.]+)\s+([\d.]+)\s+([\d.]+)\s+" + re.escape(fname) + r":(\d+)", line)
        if not m:
            continue
        ln = int(m.group(4))
        name = next((n for a, b, n in rs if a <= ln <= b), "?")
        a = acc.setdefault(name, [0.0, 0.0])
        a[0] += float(m.group(1))
        a[1] += float(m.group(2))
    for name, (i, s) in sorted(acc.items(), key=lambda x: -x[1][0]):
        print(f"{name:24s} inst {i:6.2f}%  stall-samples {s:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
