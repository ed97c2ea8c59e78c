"""Per-frame instruction and traffic constants of a step kernel from one ncu --set full capture,
written into profiles/issue_profile.json (read by bench.py for the roofline block).

    python tools/issue_profile.py gpurun_out/prof.ncu-rep cfg2/jit FRAMES_PER_LAUNCH "source note"

FRAMES_PER_LAUNCH = envs x frameskip of the captured launch.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[i], u[i]) for i, k in enumerate(h)}


def num(m, k):
    return float(m[k][0].replace(",", ""))


def main(path, key, frames, note=""):
    m = metrics(path)
    inst = num(m, "smsp__inst_executed.sum")
    thr = num(m, "smsp__thread_inst_executed.sum") if "smsp__thread_inst_executed.sum" in m else \
        num(m, "sass__thread_inst_executed_true_per_opcode")
    dur_ms = num(m, "gpu__time_duration.sum")
    unit = m["gpu__time_duration.sum"][1]
    dur_s = dur_ms / 1e3 if unit == "ms" else (dur_ms / 1e6 if unit == "us" else dur_ms / 1e9)
    clk = num(m, "sm__cycles_elapsed.avg.per_second") * 1e9
    alu_frac = num(m, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed") / 100.0
    issue = num(m, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100.0
    alu_inst = alu_frac * 148 * 4 * 0.5 * clk * dur_s
    dram = num(m, "dram__bytes_read.sum") + num(m, "dram__bytes_write.sum")
    if m["dram__bytes_read.sum"][1].startswith("M"):
        dram *= 1e6
    elif m["dram__bytes_read.sum"][1].startswith("G"):
        dram *= 1e9
    entry = {
        "warp_inst_per_frame": inst / frames,
        "thread_inst_per_frame": thr / frames,
        "threads_per_inst": thr / inst,
        "alu_inst_per_frame": alu_inst / frames,
        "alu_pipe_frac": round(alu_frac, 3),
        "issue_active": round(issue, 3),
        "dram_bytes_per_launch": dram,
        "frames_per_launch": frames,
        "source": f"{note} ({inst:.4e} warp-inst, {thr:.4e} thread-inst / {frames} frames; ALU-pipe "
                  f"warp-inst = sm__pipe_alu_cycles_active {100 * alu_frac:.1f}% of elapsed x 148 SMs x 2 per cycle)",
    }
    p = os.path.join(ROOT, "profiles", "issue_profile.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[key] = entry
    json.dump(d, open(p, "w"), indent=1)
    print(key, json.dumps(entry))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4] if len(sys.argv) > 4 else "")
