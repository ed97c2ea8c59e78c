#!/usr/bin/env python
"""Benchmark: emulated (raw) Atari frames per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--envs E] [--config cfg2|cfg3|cfg4]
    python bench.py --impl reference ...     # the CPU oracle on the host cores (reference arm)
    torchrun --nproc-per-node N bench.py --gpus N ...

Default workload (N=1): BASELINE.json configs[1] = cfg2: 4096 envs of the generated 4 KB
playfield ROM R1, frameskip 4, 84x84 grayscale max-pooled observations, random actions
(P:318-320 emulation-only load), reset-from-cache on done.  One step = one cule_step over all
envs (a0..a8 of SURVEY.md §8(a)).  Raw frames = envs x frameskip x steps.

Multi-GPU: one process per GPU, env slice [rank*E, (rank+1)*E) via env_index_base (weak
scaling); the only collective is one NCCL all_reduce of the int64[4] counters after timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (rom names, envs per GPU, frameskip, obs mode, description)
    "cfg2": (["R1"], 4096, 4, "gray84", "cfg2: 4096 envs, generated 4 KB ROM R1, fs=4, GRAY84"),
    "cfg3": (["R2"], 16384, 4, "gray84", "cfg3: 16384 envs, F8 ROM R2, fs=4, GRAY84, reset-from-cache"),
    "cfg4": (["R1", "R2", "R3", "R4"], 32768, 4, "gray84", "cfg4: 32768 envs, R1-R4 interleaved, fs=4, GRAY84"),
    # cfg5 is the whole-box configuration: 262144 envs = 32768 per GPU over 8 GPUs (run it with
    # torchrun --nproc-per-node 8 ... --config cfg5); per GPU it is the cfg4 workload
    "cfg5": (["R1", "R2", "R3", "R4"], 32768, 4, "gray84",
             "cfg5: 32768 envs per GPU (262144 on 8 GPUs), R1-R4 interleaved, fs=4, GRAY84"),
    # analysis variants (not bench lines): cfg2 with RAW observations (1 of 4 frames rendered)
    "cfg2raw": (["R1"], 4096, 4, "raw", "cfg2raw: 4096 envs, generated 4 KB ROM R1, fs=4, RAW frames"),
}

# The step kernel is bound by the integer ALU pipe (ncu: ALU pipe ~80% of its
# peak, issue ~75%): per raw frame it executes a fixed number of ALU-pipe and of all
# warp-instructions, measured once per build with ncu and committed in
# profiles/issue_profile.json (with the DRAM traffic of the same capture), keyed by config and
# engine.  achieved = that x frames per launch / the live launch time; peaks = 148 SMs x 4
# schedulers x max clock x (1/2 warp-instruction per cycle for the ALU pipe, 1 for issue).
def issue_profile(config: str, engine: str):
    try:
        with open(os.path.join(ROOT, "profiles", "issue_profile.json")) as f:
            return json.load(f).get(f"{config}/{engine}")
    except (OSError, ValueError):
        return None

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--impl", default="cule", choices=["cule", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--envs", type=int, default=0, help="override envs per GPU")
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--vtrace", type=int, default=1, choices=[0, 1],
                    help="also time the batched V-trace kernel (NEXT-3)")
    ap.add_argument("--inference-steps", type=int, default=60,
                    help="steps of the inference-path measurement (0: skip; gray84 configs only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-envs", type=int, default=16)
    ap.add_argument("--cpu-sample-steps", type=int, default=100)
    ap.add_argument("--idle-skip", type=int, default=0, choices=[0, 1],
                    help="exact idle-loop skip (off for the headline, SURVEY.md §7c.8)")
    ap.add_argument("--no-variant", action="store_true", help="skip the idle-skip-on variant run")
    ap.add_argument("--sweep", type=int, default=1, choices=[0, 1],
                    help="FPS vs num_envs sweep on R1 and on the cfg4 mix (rank 0, N=1 only)")
    ap.add_argument("--sweep-envs", default="256,1024,4096,8192,16384,32768,65536")
    ap.add_argument("--sweep-steps", type=int, default=60)
    ap.add_argument("--sweep-warmup", type=int, default=100)
    ap.add_argument("--e4", type=int, default=1, choices=[0, 1],
                    help="E4 decorrelation diagnostic (PAPER.md P:452-465; rank 0, N=1 only)")
    ap.add_argument("--window", type=int, default=100,
                    help="counter all-reduce window in steps (SURVEY.md §8(e)), on a side stream")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in open(self.path):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm = float(parts[1].split()[0])
                mx = float(parts[2].split()[0])
            except ValueError:
                continue
            sms.append(sm)
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle as it stands, on the host cores
# ---------------------------------------------------------------------------------------------
def _oracle_worker(args):
    rom_names, n_envs, fs, mode, base, steps, warmup, seed = args
    sys.path.insert(0, ROOT)
    import numpy as np
    import oracle
    from paper_1907_08467_b200.inputs import games, palette
    roms = [games.build_rom(n) for n in rom_names]
    env = oracle.OracleEnv(roms, n_envs, fs, palette.load_palette(), obs_mode=1 if mode == "gray84" else 0,
                           env_index_base=base)
    env.reset(0)
    rng = np.random.default_rng(seed)
    for _ in range(warmup):
        env.step(rng.integers(0, 18, n_envs, dtype=np.uint8))
    t0 = time.perf_counter()
    for _ in range(steps):
        env.step(rng.integers(0, 18, n_envs, dtype=np.uint8))
    dt = time.perf_counter() - t0
    return n_envs * fs * steps, dt


def oracle_fps(rom_names, fs, mode, envs_per_proc, steps, warmup, procs):
    import multiprocessing as mp
    jobs = [(rom_names, envs_per_proc, fs, mode, 1_000_000 + k * envs_per_proc, steps, warmup, 1234 + k)
            for k in range(procs)]
    t0 = time.perf_counter()
    if procs == 1:
        res = [_oracle_worker(jobs[0])]
    else:
        with mp.get_context("spawn").Pool(procs) as pool:
            res = pool.map(_oracle_worker, jobs)
    wall = time.perf_counter() - t0
    frames = sum(r[0] for r in res)
    per_proc_time = max(r[1] for r in res)
    return frames / per_proc_time, frames, per_proc_time, wall


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written), else the profiling guide's
    fallback (6.65 TB/s, 1965 MHz)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return {"hbm_gbs": float(m["hbm_gbs"]), "sm_max_mhz": float(m.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, rank, world):
    rom_names, envs, fs, mode, desc = CONFIGS[args.config]
    if args.envs:
        envs = args.envs
    if rank != 0:
        return
    cores = host_cores()
    procs = max(1, min(cores, 64))
    # each timed oracle step runs a bounded sample of the workload: `procs` processes x 4 envs
    fps, frames, t, wall = oracle_fps(rom_names, fs, mode, 4, args.steps, args.warmup, procs)
    sample = (f"{procs} oracle processes x 4 envs (global ids >= 1e6) of {desc}; "
              f"{args.warmup} warm-up + {args.steps} timed steps each")
    line = {
        "impl": "reference", "metric": "emulated frames/sec", "value": fps, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * t / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "envs_per_gpu": envs, "frameskip": fs, "obs": mode},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": procs, "kind": "oracle",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# the CUDA arm
# ---------------------------------------------------------------------------------------------
class NatureCNN:
    """The DQN/A2C Atari policy trunk (conv 8x8/4 32, 4x4/2 64, 3x3/1 64, fc 512, 18 logits),
    random init, bf16: the consumer of the frame stack for the inference-path measurement (plain
    PyTorch: the policy is not part of the emulation hot path)."""

    def __init__(self, dev):
        import torch
        g = torch.Generator(device="cpu").manual_seed(7)
        def p(*shape, fan):
            return (torch.randn(*shape, generator=g) / fan ** 0.5).to(dev, torch.bfloat16)
        self.w1, self.b1 = p(32, 4, 8, 8, fan=256), torch.zeros(32, device=dev, dtype=torch.bfloat16)
        self.w2, self.b2 = p(64, 32, 4, 4, fan=512), torch.zeros(64, device=dev, dtype=torch.bfloat16)
        self.w3, self.b3 = p(64, 64, 3, 3, fan=576), torch.zeros(64, device=dev, dtype=torch.bfloat16)
        self.w4, self.b4 = p(512, 3136, fan=3136), torch.zeros(512, device=dev, dtype=torch.bfloat16)
        self.w5, self.b5 = p(18, 512, fan=512), torch.zeros(18, device=dev, dtype=torch.bfloat16)
        # conv1 per ring position of the newest frame: input channels permuted (the frames stay in
        # place) and the 1/255 input scale folded into the weights; channels-last activations
        # (cuDNN's NHWC kernels), algorithms picked by cudnn.benchmark at the warm-up steps
        torch.backends.cudnn.benchmark = True
        self.w1s = []
        for slot in range(4):
            order = [(slot + 1 + k) % 4 for k in range(4)]  # oldest -> newest ring slots
            inv = [order.index(c) for c in range(4)]         # ring slot c holds temporal frame inv[c]
            self.w1s.append((self.w1[:, inv].float() / 255.0).to(torch.bfloat16)
                            .contiguous(memory_format=torch.channels_last))
        self.w2 = self.w2.contiguous(memory_format=torch.channels_last)
        self.w3 = self.w3.contiguous(memory_format=torch.channels_last)

    def act(self, stack, slot, gen):
        """Sample actions from the stack as the step kernel left it: slot `slot` is the newest
        frame, so conv1's input channels are permuted instead of the frames (no copy)."""
        import torch
        import torch.nn.functional as F
        x = stack.to(dtype=torch.bfloat16, memory_format=torch.channels_last)
        h = F.relu(F.conv2d(x, self.w1s[slot], self.b1, stride=4))
        h = F.relu(F.conv2d(h, self.w2, self.b2, stride=2))
        h = F.relu(F.conv2d(h, self.w3, self.b3, stride=1))
        h = F.relu(F.linear(h.flatten(1), self.w4, self.b4))
        logits = F.linear(h, self.w5, self.b5).float()
        return torch.multinomial(torch.softmax(logits, -1), 1, generator=gen).squeeze(1).to(torch.uint8)


def run_inference(env, dev, envs, world, fs, steps, rank):
    import torch

    from paper_1907_08467_b200 import dist as D
    pol = NatureCNN(dev)
    stack = env.new_stack()
    env.reset_stacked(stack, 5)
    gen = torch.Generator(device=dev)
    gen.manual_seed(77 + rank)
    slot = 0
    for t in range(3):  # warm-up (cuDNN algorithm choice)
        a = pol.act(stack, (slot - 1) % 4, gen)
        env.step_stacked(a, stack, slot)
        slot = (slot + 1) % 4
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for t in range(steps):
        a = pol.act(stack, (slot - 1) % 4, gen)
        env.step_stacked(a, stack, slot)
        slot = (slot + 1) % 4
    ev1.record()
    torch.cuda.synchronize(dev)
    ms = D.max_over_ranks(ev0.elapsed_time(ev1), device=dev)
    return {"value": envs * world * fs * steps / (ms / 1000.0), "unit": "frames/s",
            "ms_per_step": ms / steps, "steps": steps,
            "loop": "frame stack u8[N,4,84,84] written by the step kernel -> Nature-CNN policy (bf16, "
                    "random init, torch) -> device-side multinomial sampling -> next step",
            "gpu_launches_per_step": "1 emulation kernel + the policy's torch kernels"}


def run_vtrace(dev, pk):
    """Batched V-trace targets (NEXT-3, cule_vtrace): time-major fp32 [T][B], one thread per
    trajectory; a pure HBM stream of 29 bytes per (t, b) (r, V, log mu, log pi: 4 B each in,
    done 1 B in; v, rho, advantage: 4 B each out) + 4 B per bootstrap.  Timed with CUDA events
    over 50 launches replayed from one CUDA graph, inputs resident in HBM; reported at the training shape of
    the bench config (T=20 steps, B=4096) and at B=2^20 (the HBM roofline shape)."""
    import torch

    from paper_1907_08467_b200.vtrace import vtrace
    out = {}
    for T, B in ((20, 4096), (20, 1 << 20)):
        g = torch.Generator(device=dev)
        g.manual_seed(3)
        r = torch.randn(T, B, device=dev, generator=g)
        V = torch.randn(T, B, device=dev, generator=g)
        vb = torch.randn(B, device=dev, generator=g)
        lm = torch.randn(T, B, device=dev, generator=g) * 0.5
        lp = torch.randn(T, B, device=dev, generator=g) * 0.5
        d = (torch.rand(T, B, device=dev, generator=g) < 0.05).to(torch.uint8)
        bufs = (torch.empty_like(r), torch.empty_like(r), torch.empty_like(r))
        side = torch.cuda.Stream(dev)
        with torch.cuda.stream(side):
            for _ in range(3):
                vtrace(r, V, vb, lm, lp, d, 0.99, out=bufs)
        torch.cuda.synchronize(dev)
        # 50 launches captured in one CUDA graph: the kernel's own time, not the host's call rate
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            for _ in range(50):
                vtrace(r, V, vb, lm, lp, d, 0.99, out=bufs)
        graph.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize(dev)
        s = e0.elapsed_time(e1) / 1000.0 / 50
        nbytes = T * B * 29 + 4 * B
        out[f"T{T}_B{B}"] = {"us_per_launch": s * 1e6, "achieved_gbs": nbytes / s / 1e9,
                             "frac_hbm": nbytes / s / 1e9 / pk["hbm_gbs"], "bytes_per_launch": nbytes,
                             "trajectories_per_s": B / s}
    out["roofline"] = {"bound": "hbm", "peak_gbs": pk["hbm_gbs"], "peak_source": pk["source"]}
    return out


def time_steps(env, acts, t0, K, stream):
    """Device time (ms) of K steps acts[t0:t0+K] on `stream` (CUDA events, sync on both sides)."""
    import torch
    torch.cuda.synchronize(env.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for t in range(t0, t0 + K):
        env.step(acts[t])
    e1.record(stream)
    torch.cuda.synchronize(env.device)
    return e0.elapsed_time(e1)


def run_sweep(dev, args, stream):
    """Emulated FPS vs num_envs (BASELINE.json metric "... vs num_envs"; SURVEY.md §8(d) sweep):
    R1 alone and the cfg4 mix (R1-R4 interleaved), fs=4, GRAY84, random actions; each point
    warms up `sweep_warmup` steps and times `sweep_steps`; the engine the library chose is named."""
    import torch

    from paper_1907_08467_b200 import Env
    from paper_1907_08467_b200.inputs import games
    out = {"steps": args.sweep_steps, "warmup": args.sweep_warmup, "fs": 4, "obs": "gray84", "points": {}}
    W, K = args.sweep_warmup, args.sweep_steps
    for label, names in (("R1", ["R1"]), ("cfg4_mix", ["R1", "R2", "R3", "R4"])):
        roms = [games.build_rom(n) for n in names]
        pts = []
        for n in [int(x) for x in args.sweep_envs.split(",") if x]:
            env = Env(roms, n, 4, device=dev)
            env.reset(0)
            gen = torch.Generator(device=dev)
            gen.manual_seed(99)
            acts = torch.randint(0, 18, (W + K, n), generator=gen, device=dev, dtype=torch.uint8)
            for t in range(W):
                env.step(acts[t])
            ms = time_steps(env, acts, W, K, stream)
            pts.append({"envs": n, "fps": n * 4 * K / (ms / 1000.0), "ms_per_step": ms / K, "engine": env.engine})
            env.close()
            del acts
        out["points"][label] = pts
    return out


def run_e4(dev, stream, n_list=(512, 32768), steps=300, window=10):
    """E4 decorrelation diagnostic: every env starts from ONE
    cache entry (cule_set_state), random actions; FPS per 10-step window and the resets in each
    window.  Identical envs start converged (no divergence) and decorrelate as random actions and
    resets spread them, which is what the W = 200 warm-up of the bench skips."""
    import numpy as np
    import torch

    from paper_1907_08467_b200 import Env
    from paper_1907_08467_b200.inputs import games
    rom = games.build_rom("R1")
    out = {"rom": "R1", "fs": 4, "obs": "gray84", "window_steps": window, "runs": {}}
    for n in n_list:
        env = Env([rom], n, 4, device=dev)
        env.reset(0)
        st = env.get_state()
        machine = np.r_[0:61, 64:192]
        st[:, machine] = st[0, machine]          # every env = env 0's cache entry (same ROM)
        env.set_state(st)
        gen = torch.Generator(device=dev)
        gen.manual_seed(5)
        acts = torch.randint(0, 18, (steps, n), generator=gen, device=dev, dtype=torch.uint8)
        fps, resets = [], []
        for w0 in range(0, steps, window):
            done_sum = torch.zeros((), dtype=torch.int64, device=dev)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for t in range(w0, w0 + window):
                _, _, d = env.step(acts[t])
                done_sum += d.sum()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1)
            fps.append(n * 4 * window / (ms / 1000.0))
            resets.append(int(done_sum.item()))
        out["runs"][str(n)] = {"engine": env.engine, "fps_per_window": fps, "resets_per_window": resets,
                               "first_window_fps": fps[0], "last_10_windows_mean_fps": sum(fps[-10:]) / 10}
        env.close()
    out["note"] = ("the done-count reduction (torch) runs inside each window; it is the same for every window")
    return out


def oracle_single_core(rom_names, fs, mode):
    """SURVEY.md §8(d) oracle baseline: FPS_1 = the oracle on ONE core (R1, fs=4, GRAY84, 64 envs
    x 50 steps) and the cfg1 oracle wall time (16 envs x 100 frames, fs=1, RAW)."""
    import numpy as np
    import oracle
    from paper_1907_08467_b200.inputs import games, palette
    rom = games.build_rom("R1")
    pal = palette.load_palette()
    env = oracle.OracleEnv([rom], 64, 4, pal, obs_mode=1)
    env.reset(0)
    rng = np.random.default_rng(1234)
    t0 = time.perf_counter()
    for _ in range(50):
        env.step(rng.integers(0, 18, 64, dtype=np.uint8))
    dt = time.perf_counter() - t0
    env.close()
    t1 = time.perf_counter()
    env = oracle.OracleEnv([rom], 16, 1, pal, obs_mode=0)
    env.reset(0)
    for _ in range(100):
        env.step(rng.integers(0, 18, 16, dtype=np.uint8))
    cfg1_wall = time.perf_counter() - t1
    env.close()
    return {"fps_1core": 64 * 4 * 50 / dt, "fps_1core_sample": "R1, fs=4, GRAY84, 64 envs x 50 steps, 1 process",
            "cfg1_oracle_wall_s": cfg1_wall,
            "cfg1_sample": "16 envs x 100 frames, fs=1, RAW (reset-cache build included)"}


def run_cule(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1907_08467_b200 import Env, build
    from paper_1907_08467_b200 import dist as D
    from paper_1907_08467_b200.inputs import games

    if local_rank == 0:
        build.build()          # one build per node, before any rank loads the library
    if world > 1:
        dist.barrier()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    rom_names, envs, fs, mode, desc = CONFIGS[args.config]
    if args.envs:
        envs = args.envs
    roms = [games.build_rom(n) for n in rom_names]
    base, _ = D.shard(envs, rank)
    env = Env(roms, envs, fs, obs_mode=mode, env_index_base=base, device=dev, idle_skip=args.idle_skip)
    stream = torch.cuda.current_stream(dev)
    env.reset(0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    W, K = args.warmup, args.steps
    acts = torch.randint(0, 18, (W + K, envs), generator=gen, device=dev, dtype=torch.uint8)
    for t in range(W):
        env.step(acts[t])
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    # once per reporting window the int64[4] counters are copied on the step
    # stream and all-reduced (NCCL, N > 1) on a side stream that waits only for that copy, so the
    # collective never blocks the step stream
    side = torch.cuda.Stream(dev)
    win_bufs, win_works = [], []
    ev0.record(stream)
    for t in range(W, W + K):
        env.step(acts[t])
        if args.window > 0 and (t - W + 1) % args.window == 0:
            buf = torch.empty(4, dtype=torch.int64, device=dev)
            env.counters_into(buf)
            ready = torch.cuda.Event()
            ready.record(stream)
            side.wait_event(ready)
            with torch.cuda.stream(side):
                buf.record_stream(side)
                if world > 1:
                    win_works.append(dist.all_reduce(buf, op=dist.ReduceOp.SUM, async_op=True))
            win_bufs.append(buf)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    for w in win_works:
        w.wait()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    windows = [[int(x) for x in b.cpu().tolist()] for b in win_bufs]
    ms = ev0.elapsed_time(ev1)
    ms_max = D.max_over_ranks(ms, device=dev)
    counters = D.reduce_counters(env.counters())
    frames_total = envs * world * fs * K
    fps = frames_total / (ms_max / 1000.0)

    # e2e through the C-ABI with pinned HOST buffers: H2D actions, step, D2H obs/rewards/dones
    ob = env.obs_bytes
    h_act = torch.zeros(envs, dtype=torch.uint8).pin_memory()
    h_obs = torch.zeros((envs, ob), dtype=torch.uint8).pin_memory()
    h_rew = torch.zeros(envs, dtype=torch.int32).pin_memory()
    h_done = torch.zeros(envs, dtype=torch.uint8).pin_memory()
    hgen = torch.Generator()
    hgen.manual_seed(4321 + rank)
    host_acts = torch.randint(0, 18, (args.e2e_steps + 3, envs), generator=hgen, dtype=torch.uint8)
    for t in range(3):
        h_act.copy_(host_acts[t])
        env.step_host(h_act, h_obs, h_rew, h_done)
    if world > 1:
        dist.barrier()
    e0 = time.perf_counter()
    for t in range(args.e2e_steps):
        h_act.copy_(host_acts[t])
        env.step_host(h_act, h_obs, h_rew, h_done)
    e_dt = D.max_over_ranks(time.perf_counter() - e0, device=dev)
    e2e_fps = envs * world * fs * args.e2e_steps / e_dt

    # variant (not the headline): the same workload with the exact idle-loop skip
    variant = None
    if not args.no_variant and not args.idle_skip and world == 1:
        env2 = Env(roms, envs, fs, obs_mode=mode, env_index_base=base, device=dev, idle_skip=1)
        env2.reset(0)
        for t in range(W):
            env2.step(acts[t])
        torch.cuda.synchronize(dev)
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        for t in range(W, W + K):
            env2.step(acts[t])
        v1.record(stream)
        torch.cuda.synchronize(dev)
        vms = v0.elapsed_time(v1)
        variant = {"idle_skip": 1, "value": envs * fs * K / (vms / 1000.0), "unit": "frames/s",
                   "ms_per_step": vms / K, "note": "exact closed-form skip of [timer read; branch back] "
                                                   "poll loops (DESIGN.md §2 R#24); reported beside the "
                                                   "headline, never as it"}
        env2.close()

    # inference path: frame stack written by the step kernel, a small
    # random-init policy reading it in place, device-side action sampling; emulated frames/s
    inference = None
    if args.inference_steps > 0 and mode == "gray84" and not args.envs:
        inference = run_inference(env, dev, envs, world, fs, args.inference_steps, rank)

    if rank != 0:
        return
    # roofline of the dominant (only) kernel: the step kernel, one launch per step
    pk = peaks()
    launch_s = ms_max / 1000.0 / K
    alg_bytes_per_env = 208 * 2 + 1 + 4 + 1 + (7056 if mode == "gray84" else 33600)
    alg_bytes = alg_bytes_per_env * envs
    hbm_gbs = alg_bytes / launch_s / 1e9
    sm_mhz = clk.get("sm_mhz") or pk["sm_max_mhz"]
    issue_peak = 148 * 4 * pk["sm_max_mhz"] * 1e6 / 1e12  # T warp-instr/s at max clock
    alu_peak = issue_peak / 2.0  # the integer ALU pipe takes a warp-instruction every 2 cycles per SMSP
    prof = issue_profile(args.config, env.engine) if not args.envs else None
    ipf = prof["warp_inst_per_frame"] if prof else None
    apf = prof.get("alu_inst_per_frame") if prof else None
    issue = {"unit": "Twarp-inst/s", "peak": issue_peak,
             "achieved": (ipf * envs * fs / launch_s / 1e12) if ipf else None}
    issue["frac"] = issue["achieved"] / issue_peak if issue["achieved"] else None
    # lane-level issue: thread-instructions per second against 32 lanes per issue slot
    tpf = prof.get("thread_inst_per_frame") if prof else None
    lane_peak = issue_peak * 32.0
    lane = {"unit": "Tthread-inst/s", "peak": lane_peak,
            "achieved": (tpf * envs * fs / launch_s / 1e12) if tpf else None,
            "threads_per_warp_inst": prof.get("threads_per_inst") if prof else None}
    lane["frac"] = lane["achieved"] / lane_peak if lane["achieved"] else None
    roof = {"bound": "alu", "unit": "Twarp-inst/s (integer ALU pipe)", "peak": alu_peak,
            "achieved": (apf * envs * fs / launch_s / 1e12) if apf else None,
            "issue": issue,
            "lane_issue": lane,
            "traffic": prof["dram_bytes_per_launch"] if prof else None,
            "traffic_over_algorithmic": (prof["dram_bytes_per_launch"] / alg_bytes) if prof else None,
            "profile": prof["source"] if prof else None,
            "alu_pipe_frac_ncu": prof.get("alu_pipe_frac") if prof else None,
            "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": pk["hbm_gbs"], "frac": hbm_gbs / pk["hbm_gbs"],
                    "alg_bytes_per_launch": alg_bytes,
                    "note": "north_star's HBM fraction for state-plus-frame traffic: algorithmic bytes "
                            "(2x208 state + 6 action/reward/done + observation per env-step) / launch time"},
            "peak_source": pk["source"] + "; ALU and issue peaks from 148 SMs x 4 SMSPs x max SM clock"}
    roof["frac"] = roof["achieved"] / alu_peak if roof["achieved"] else None
    line = {
        "metric": "emulated frames/sec", "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": desc, "envs_per_gpu": envs, "frameskip": fs, "obs": mode,
                   "actions": "uniform random over 18, torch cuda generator seed 1234+rank",
                   "l2": ("per-step working set vs 126 MB L2: staged gray frames " +
                          f"{envs * 33600 * (1 if env.engine in ('jit', 'scalar') else 2) / 1e6:.0f} MB "
                          "(frame fs-1 for the one-env-per-warp engines jit/scalar; fs-1 and fs for "
                          "vjit/simt) + obs " +
                          f"{envs * (7056 if mode == 'gray84' else 33600) / 1e6:.0f} MB + state " +
                          f"{envs * 256 / 1e6:.0f} MB; no flush between steps"),
                   "parallelism": f"dp{world} (env shards)", "engine": env.engine},
        "fps_per_env": fps / (envs * world),
        "training_frames_per_s": fps / 4,
        "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": envs,
                "d2h_bytes_per_step": envs * (ob + 4 + 1)},
        "gpu_launches": K,
        "inference": inference,
        "variant": variant,
        "roofline": roof,
        "clocks": clk,
        "counters": {"frames": int(counters[0]), "episodes": int(counters[1]),
                     "return_sum": int(counters[2]), "faults": int(counters[3])},
        "counter_windows": {"every_steps": args.window, "reduced_over_ranks": world > 1,
                            "side_stream": True, "cumulative": windows},
    }
    if args.vtrace:
        line["vtrace"] = run_vtrace(dev, pk)
    env.close()
    if args.sweep and world == 1 and not args.envs:
        line["sweep"] = run_sweep(dev, args, stream)
    if args.e4 and world == 1 and not args.envs:
        line["e4"] = run_e4(dev, stream)
    if not args.no_cpu_baseline and world == 1:
        cores = host_cores()
        procs = max(1, min(cores, 64))
        cfps, frames, t, wall = oracle_fps(rom_names, fs, mode, args.cpu_sample_envs,
                                           args.cpu_sample_steps, 2, procs)
        line["cpu_baseline"] = {"value": cfps, "unit": "frames/s", "cores": procs, "kind": "oracle",
                                "sample": f"{procs} processes x {args.cpu_sample_envs} envs x "
                                          f"{args.cpu_sample_steps} steps of {desc} ({frames} frames, "
                                          f"{t:.1f} s)", "cpu": cpu_model()}
        line["cpu_baseline"].update(oracle_single_core(rom_names, fs, mode))
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        pass
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # NCCL's INIT lines (ranks, communicator) stay visible on stderr for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_cule(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
