"""Aggregate ncu per-instruction counters by CUDA source line (builds use -lineinfo).

    python tools/ncu_source.py gpurun_out/prof.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = {}
    cur_file, cur_line, cur_src = "?", None, ""
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] == "Function Name":
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None:
            continue
        if row[0] and row[0].isdigit():
            cur_line, cur_src = int(row[0]), row[1].strip()
            if row[2] == "-":
                continue
        if cur_line is None:
            continue
        d = dict(zip(hdr[2:], row[2:]))
        try:
            ie = float(d.get("Instructions Executed", 0) or 0)
            te = float(d.get("Thread Instructions Executed", 0) or 0)
            sm = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        except ValueError:
            continue
        k = (cur_file, cur_line)
        a = agg.setdefault(k, [0.0, 0.0, 0.0, cur_src])
        a[0] += ie
        a[1] += te
        a[2] += sm
    tot = sum(v[0] for v in agg.values()) or 1
    tots = sum(v[2] for v in agg.values()) or 1
    print(f"total warp instructions {tot:.4e}; stall samples {tots:.0f}")
    print(f"{'inst%':>6} {'samp%':>6} {'thr/inst':>8}  location")
    for (f, ln), (ie, te, sm, src) in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
        print(f"{100 * ie / tot:6.2f} {100 * sm / tots:6.2f} {te / max(ie, 1):8.1f}  {f}:{ln}  {src[:90]}")
    by_file = {}
    for (f, ln), v in agg.items():
        b = by_file.setdefault(f, [0.0, 0.0])
        b[0] += v[0]
        b[1] += v[2]
    print("--- by file")
    for f, (ie, sm) in sorted(by_file.items(), key=lambda kv: -kv[1][1]):
        print(f"{100 * ie / tot:6.2f} {100 * sm / tots:6.2f}  {f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
