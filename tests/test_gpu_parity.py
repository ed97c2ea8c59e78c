"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle, bit-exact.

Every comparison is element by element on the same seeded inputs: observations, rewards,
dones and the full 256-byte per-env snapshot (SURVEY.md §8(c).14 "Batched == sequential").
"""
import numpy as np
import pytest

import helpers as H
from paper_1907_08467_b200.inputs import games, micro

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True, params=["simt", "scalar", "jit", "vjit", "wsvjit"])
def engine(request, monkeypatch):
    """Every parity test runs on all four engines: the batched SIMT datapath, the scalar engine
    (one env per warp, record-driven interpreter, warp-cooperative TIA replay), the JIT
    engine (the scalar engine with the cartridge code translated to CUDA, csrc/jit.h) and the
    VJIT engine (one env per lane running the translated code, block-scheduled by warp vote,
    csrc/vjit_kernels.cuh) and its warp-specialized variant WSVJIT (producer warps emulate,
    consumer warps render)."""
    monkeypatch.setenv("CULE_ENGINE", request.param)
    return request.param


def skip_jit_debug(engine):
    if engine in ("jit", "vjit", "wsvjit"):
        pytest.skip("debug-entry test: the translated engines' debug_exec runs an interpreter (tested as "
                    "'scalar' / 'simt')")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1907_08467_b200 import build
    build.build()
    import oracle
    oracle.build()


def check_engine(gpu):
    """The engine the fixture asked for is the one that runs (the scalar engine needs its
    pre-decoded records to fit in shared memory; a silent fallback would hide it from tests)."""
    import os
    want = os.environ.get("CULE_ENGINE")
    assert gpu.engine == want, f"asked for the {want} engine, got {gpu.engine}"


def pair(roms, n, fs, mode="gray84", **cfg):
    import oracle
    from paper_1907_08467_b200 import Env
    gpu = Env(roms, n, fs, obs_mode=mode, **cfg)
    check_engine(gpu)
    ref = oracle.OracleEnv(roms, n, fs, H.palette_rgb(), obs_mode=1 if mode == "gray84" else 0, **cfg)
    return gpu, ref


def assert_same_state(gs, rs, what=""):
    if not (gs == rs).all():
        bad = np.nonzero((gs != rs).any(1))[0]
        i = int(bad[0])
        cols = np.nonzero(gs[i] != rs[i])[0]
        raise AssertionError(f"{what}: {len(bad)} envs differ; env {i} bytes {cols[:16].tolist()} "
                             f"gpu {gs[i][cols[:16]].tolist()} oracle {rs[i][cols[:16]].tolist()}")


def run_parity(gpu, ref, steps, seed=1234, reset_seed=0, check_every=1):
    og = gpu.reset(reset_seed).cpu().numpy()
    orf = ref.reset(reset_seed)
    assert (og == orf).all(), "reset observations differ"
    assert_same_state(gpu.get_state(), ref.get_state(), "after reset")
    acts = H.random_actions(gpu.num_envs, steps, seed)
    n_done = 0
    for t in range(steps):
        a = torch.from_numpy(acts[t]).to(gpu.device)
        o, r, d = gpu.step(a)
        o2, r2, d2 = ref.step(acts[t])
        o, r, d = o.cpu().numpy(), r.cpu().numpy(), d.cpu().numpy()
        assert (r == r2).all(), f"step {t}: rewards differ"
        assert (d == d2).all(), f"step {t}: dones differ"
        if not (o == o2).all():
            bad = np.nonzero((o != o2).reshape(len(o), -1).any(1))[0]
            raise AssertionError(f"step {t}: observations differ for envs {bad[:8].tolist()}")
        if t % check_every == 0 or t == steps - 1:
            assert_same_state(gpu.get_state(), ref.get_state(), f"step {t}")
        n_done += int(d.sum())
    c = gpu.counters().cpu().numpy()
    assert (c == ref.counters()).all(), (c, ref.counters())
    return n_done


def test_cfg1_raw_16x100():
    """SURVEY.md §7(b) minimum slice: R1, 16 envs, fs=1, RAW, 100 frames, everything compared."""
    gpu, ref = pair([games.build_rom("R1")], 16, 1, "raw", reset_cache_size=30)
    run_parity(gpu, ref, 100)


@pytest.mark.parametrize("name", ["R1", "R2", "R3", "R4"])
def test_gray84_fs4(name):
    gpu, ref = pair([games.build_rom(name)], 200, 4, reset_cache_size=8)
    run_parity(gpu, ref, 40, check_every=5)


def test_mixed_roms_ragged():
    roms = [games.build_rom(n) for n in ("R1", "R2", "R3", "R4")]
    gpu, ref = pair(roms, 131, 4, reset_cache_size=6)
    run_parity(gpu, ref, 30, check_every=10)


@pytest.mark.parametrize("epw", ["1", "4", "32"])
def test_launch_shape_independence(epw, monkeypatch):
    """Results do not depend on the launch shape: envs per warp (CULE_EPW; CULE_VEPW for the
    VJIT engine), block size and the ROM-grouped env-to-lane permutation (S:283-286
    worker-count independence)."""
    monkeypatch.setenv("CULE_EPW", epw)
    monkeypatch.setenv("CULE_VEPW", epw)
    monkeypatch.setenv("CULE_BLOCK", "64")
    monkeypatch.setenv("CULE_VWPB", "2")
    roms = [games.build_rom(n) for n in ("R1", "R3", "R2")]
    gpu, ref = pair(roms, 77, 4, reset_cache_size=4, env_index_base=5)
    run_parity(gpu, ref, 12, check_every=4)


def test_raw_fs4_and_fs2():
    gpu, ref = pair([games.build_rom("R2")], 40, 4, "raw", reset_cache_size=4)
    run_parity(gpu, ref, 20, check_every=4)
    gpu, ref = pair([games.build_rom("R3")], 40, 2, "gray84", reset_cache_size=4)
    run_parity(gpu, ref, 20, check_every=4)


def test_episode_ends_and_resets():
    # short episode cap forces done + reset-from-cache inside the window (cfg3 behaviour)
    gpu, ref = pair([games.build_rom("R1"), games.build_rom("R3")], 96, 4,
                    reset_cache_size=5, max_episode_frames=24)
    n_done = run_parity(gpu, ref, 25, check_every=3)
    assert n_done > 96


@pytest.mark.parametrize("src", [micro.m17_score(), micro.m14_jam(100), micro.m15_no_vsync(100),
                                 micro.m20_timer_polls(), micro.m21_timint_spin(100)])
def test_micro_programs_env(src):
    rom = micro.build(src)
    gpu, ref = pair([rom, games.build_rom("R1")], 34, 4, reset_cache_size=3, max_random_frames=2)
    og = gpu.reset(0)
    ref.reset(0)
    for t in range(40):
        a = np.full(34, 1 if t % 3 else 0, np.uint8)
        o, r, d = gpu.step(torch.from_numpy(a).cuda())
        o2, r2, d2 = ref.step(a)
        assert (r.cpu().numpy() == r2).all() and (d.cpu().numpy() == d2).all(), t
        assert (o.cpu().numpy() == o2).all(), t
        assert_same_state(gpu.get_state(), ref.get_state(), f"step {t}")
    assert (gpu.counters().cpu().numpy() == ref.counters()).all()


STATIC_CASES = [
    dict(pokes=[(0x09, 0x1E), (0x08, 0x44), (0x0E, 0xA5), (0x0A, 1)]),
    dict(pokes=[(0x06, 0x86), (0x1B, 0xC1), (0x04, 7)], positions=[(0x10, 20)], hmove=True),
    dict(pokes=[(0x1B, 0xFF), (0x1F, 2), (0x0A, 0x35), (0x0F, 0xFF)],
         positions=[(0x10, 20), (0x14, 21)], store_collisions=True),
    dict(pokes=[(0x09, 0x1E), (0x20, 0x70)], positions=[(0x10, 3)], hmove_row0=True),
    dict(pokes=[(0x1B, 0xFF), (0x1C, 0x81), (0x1D, 2), (0x1E, 2), (0x25, 1), (0x05, 0x33)],
         positions=[(0x10, 12), (0x11, 14), (0x12, 13), (0x13, 30)], store_collisions=True),
]


@pytest.mark.parametrize("case", range(len(STATIC_CASES)))
def test_static_frames_raw(case):
    rom = micro.build(micro.static_frame(**STATIC_CASES[case]))
    gpu, ref = pair([rom], 8, 1, "raw", reset_cache_size=2, max_random_frames=1)
    run_parity(gpu, ref, 6)


def _random_states(n, n_roms, rng, banks=None):
    """Valid random snapshots (canonical field ranges) for single-instruction
    cross-checks."""
    s = np.zeros((n, 256), np.uint8)
    s[:, 0:4] = rng.integers(0, 256, (n, 4))
    s[:, 4] = (rng.integers(0, 256, n) & ~0x10) | 0x20
    rom_id = rng.integers(0, n_roms, n)
    s[:, 61] = rom_id
    if banks is None:
        s[:, 5] = np.where(rom_id >= 2, rng.integers(0, 2, n), 0)     # ROMs 2,3 are F8
    else:                                                             # banks of each ROM
        s[:, 5] = (rng.integers(0, 8, n) % np.asarray(banks)[rom_id]).astype(np.uint8)
    pcs = np.where(rng.random(n) < 0.9, rng.integers(0xF000, 0x10000, n),
                   rng.integers(0x80, 0x100, n))
    pcs = np.where(rng.random(n) < 0.02, rng.integers(0, 0x10000, n), pcs)
    s[:, 6] = pcs & 0xFF
    s[:, 7] = pcs >> 8
    fc = rng.integers(0, 76 * 300, n)
    s[:, 8:12] = fc.astype("<u4").view(np.uint8).reshape(n, 4)
    tS = rng.choice([0, 3, 6, 10], n)
    tV = rng.integers(0, 256, n)
    e = rng.integers(0, (tV.astype(np.int64) << tS) + 300)
    s[:, 12:16] = (fc - e).astype("<i4").view(np.uint8).reshape(n, 4)
    s[:, 16] = tV
    s[:, 17] = tS
    s[:, 18] = rng.integers(0, 256, n)
    s[:, 19] = rng.choice([0, 0x80], n)
    coll = rng.integers(0, 1 << 16, n) & ~(1 << 13)
    s[:, 20] = coll & 0xFF
    s[:, 21] = coll >> 8
    comb = np.where(rng.random(n) < 0.5, -1, rng.integers(0, 300, n))
    s[:, 22:24] = comb.astype("<i2").view(np.uint8).reshape(n, 2)
    for off in (24, 25, 33, 34, 42, 43, 44, 45, 51, 52, 53, 54, 55):
        s[:, off] = rng.integers(0, 2, n)
    for off in (26, 27, 28, 29, 30, 31, 32, 35, 36, 37, 38, 39, 40, 41):
        s[:, off] = rng.integers(0, 256, n)
    for off in (46, 47, 48, 49, 50):
        s[:, off] = rng.integers(0, 16, n)
    for off in range(56, 61):
        s[:, off] = rng.integers(0, 160, n)
    s[:, 64:192] = rng.integers(0, 256, (n, 128))
    return s


@pytest.mark.parametrize("n_instr", [1, 3, 40])
def test_random_instructions(n_instr, engine):
    """>= 1e5 random (opcode, registers, memory) cases through the debug entry of the kernel
    against the oracle's single-instruction execution.  Random ROM bytes put
    every opcode, addressing mode and operand at every offset, so the scalar engine's
    pre-decoded fast classes and their edge cases (window-crossing branches, jumps into other
    windows, zero-page indexing into the TIA, RAM-based abs,Y page crosses, F8 hotspots, code
    in RAM) are all exercised.  Two 4 KB + one F8 ROM for the scalar engine (its records must fit
    in shared memory), two of each for the batched engine."""
    skip_jit_debug(engine)
    import oracle
    from paper_1907_08467_b200 import Env
    rng = np.random.default_rng(100 + n_instr)
    n_f8 = 1 if engine == "scalar" else 2
    roms = [rng.integers(0, 256, 4096, dtype=np.uint8).tobytes() for _ in range(2)] + \
           [rng.integers(0, 256, 8192, dtype=np.uint8).tobytes() for _ in range(n_f8)]
    n = 100_000 if n_instr == 1 else 20_000
    # RAW mode: no palette needed; only the debug entry is used (K=1 cache, 0 frames)
    gpu = Env(roms, n, 1, obs_mode="raw", reset_cache_size=1, startup_frames=0, max_random_frames=0)
    check_engine(gpu)
    st = _random_states(n, len(roms), rng)
    gpu.set_state(st)
    status = gpu.debug_exec(n_instr).cpu().numpy()
    got = gpu.get_state()
    bad = []
    for i in range(n):
        s = st[i].copy()
        r, _ = oracle.exec_instr(roms[st[i, 61]], s, n_instr)
        if r != status[i] or not (s == got[i]).all():
            bad.append(i)
            if len(bad) > 5:
                break
    if bad:
        i = bad[0]
        s = st[i].copy()
        r, _ = oracle.exec_instr(roms[st[i, 61]], s, n_instr)
        cols = np.nonzero(s != got[i])[0]
        op = roms[st[i, 61]][(int(st[i, 5]) << 12) + (H.pc(st[i]) & 0xFFF)] if H.pc(st[i]) & 0x1000 else None
        raise AssertionError(f"{len(bad)}+ mismatches; env {i} op {op} pc {H.pc(st[i]):04x} status "
                             f"gpu {status[i]} oracle {r}; bytes {cols.tolist()[:12]} gpu "
                             f"{got[i][cols].tolist()[:12]} oracle {s[cols].tolist()[:12]}")


@pytest.mark.parametrize("n_instr", [1, 40])
def test_mapper_random_instructions(n_instr, engine):
    """NEXT-4 mappers: random instructions on random 2K / F6 / F4 cartridges (hotspots at
    $1FF6-$1FF9 and $1FF4-$1FFB, the 2K mirror) through the debug entry, against the oracle.
    The scalar engine takes 2K + F6 (its records must fit in shared memory); F4 runs on the
    batched engine."""
    skip_jit_debug(engine)
    import oracle
    from paper_1907_08467_b200 import Env
    rng = np.random.default_rng(500 + n_instr)
    sizes = [2048, 16384] if engine == "scalar" else [2048, 16384, 32768]
    roms = [rng.integers(0, 256, n, dtype=np.uint8).tobytes() for n in sizes]
    banks = [max(1, n // 4096) for n in sizes]
    n = 60_000 if n_instr == 1 else 12_000
    gpu = Env(roms, n, 1, obs_mode="raw", reset_cache_size=1, startup_frames=0, max_random_frames=0)
    check_engine(gpu)
    st = _random_states(n, len(roms), rng, banks)
    gpu.set_state(st)
    status = gpu.debug_exec(n_instr).cpu().numpy()
    got = gpu.get_state()
    bad = []
    for i in range(n):
        s = st[i].copy()
        r, _ = oracle.exec_instr(roms[st[i, 61]], s, n_instr)
        if r != status[i] or not (s == got[i]).all():
            bad.append(i)
            if len(bad) > 5:
                break
    assert not bad, f"{len(bad)}+ mismatches, first env {bad[0]} rom {st[bad[0], 61]} pc {H.pc(st[bad[0]]):04x}"


@pytest.mark.parametrize("nbanks", [4, 8])
def test_m22_bank_programs(nbanks, engine):
    """The F6 / F4 micro-programs (oracle pins in test_oracle_riot_cart.py) give the same state
    on the GPU after every step of 37 instructions."""
    skip_jit_debug(engine)
    import oracle
    from paper_1907_08467_b200 import Env
    if engine == "scalar" and nbanks == 8:
        pytest.skip("F4 records do not fit the scalar engine's shared memory (batched engine runs it)")
    rom = micro.build(micro.m22_banks(nbanks), 4096 * nbanks)
    gpu = Env([rom], 3, 1, obs_mode="raw", reset_cache_size=1, startup_frames=0, max_random_frames=0)
    check_engine(gpu)
    s0 = np.stack([oracle.power_on(rom)] * 3)
    gpu.set_state(s0)
    for _ in range(10):
        gpu.debug_exec(37)
        for i in range(3):
            oracle.exec_instr(rom, s0[i], 37)
        assert_same_state(gpu.get_state(), s0, "m22")


def test_set_state_windowed_parity():
    """Late, decorrelated states: run the oracle 30 steps, load its snapshots into the GPU, and
    compare 10 more steps (SURVEY.md §8(d) windowed parity)."""
    gpu, ref = pair([games.build_rom("R1"), games.build_rom("R2")], 64, 4, reset_cache_size=5)
    gpu.reset(3)
    ref.reset(3)
    acts = H.random_actions(64, 40, 77)
    for t in range(30):
        ref.step(acts[t])
    gpu.set_state(ref.get_state())
    assert_same_state(gpu.get_state(), ref.get_state(), "set_state round trip")
    for t in range(30, 40):
        o, r, d = gpu.step(torch.from_numpy(acts[t]).cuda())
        o2, r2, d2 = ref.step(acts[t])
        assert (o.cpu().numpy() == o2).all() and (r.cpu().numpy() == r2).all()
        assert_same_state(gpu.get_state(), ref.get_state(), f"step {t}")


def test_num_envs_and_step_host_equivalence():
    from paper_1907_08467_b200 import Env
    rom = games.build_rom("R1")
    big = Env([rom], 300, 4, reset_cache_size=6)
    small = Env([rom], 20, 4, reset_cache_size=6)
    host = Env([rom], 20, 4, reset_cache_size=6)
    for e in (big, small, host):
        check_engine(e)
    big.reset(9)
    small.reset(9)
    host.reset(9)
    acts = H.random_actions(300, 15, 5)
    h_act = torch.zeros(20, dtype=torch.uint8).pin_memory()
    h_obs = torch.zeros((20, 84, 84), dtype=torch.uint8).pin_memory()
    h_rew = torch.zeros(20, dtype=torch.int32).pin_memory()
    h_done = torch.zeros(20, dtype=torch.uint8).pin_memory()
    for t in range(15):
        ob, rb, db = big.step(torch.from_numpy(acts[t]).cuda())
        os_, rs, ds = small.step(torch.from_numpy(acts[t, :20]).cuda())
        h_act.copy_(torch.from_numpy(acts[t, :20]))
        host.step_host(h_act, h_obs, h_rew, h_done)
        assert (ob[:20] == os_).all() and (rb[:20] == rs).all() and (db[:20] == ds).all()
        assert (h_obs == os_.cpu()).all() and (h_rew == rs.cpu()).all() and (h_done == ds.cpu()).all()
    assert (big.get_state()[:20] == small.get_state()).all()


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4"])
def test_sampled_parity_at_full_size(cfg):
    """cfg3 (16384 envs, F8 ROM R2) and cfg4 (32768 envs, R1-R4 interleaved) at full size in the
    bench's launch configuration (default envs-per-warp heuristic, ROM-grouped lanes); sampled
    envs replayed in the oracle with their global ids, including the last env (ragged tail)."""
    import oracle
    from paper_1907_08467_b200 import Env
    names, N = (["R2"], 16384) if cfg == "cfg3" else (["R1", "R2", "R3", "R4"], 32768)
    roms = [games.build_rom(n) for n in names]
    steps = 8
    gpu = Env(roms, N, 4)
    check_engine(gpu)
    gpu.reset(0)
    acts = H.random_actions(N, steps, 99)
    rng = np.random.default_rng(1)
    sample = np.unique(np.concatenate([np.arange(0, 9), [N // 2 - 1, N // 2, N - 2, N - 1],
                                       rng.integers(0, N, 19)]))
    ref = oracle.OracleEnv(roms, len(sample), 4, H.palette_rgb())
    ref.set_env_ids(sample)
    ref.reset(0)
    for t in range(steps):
        o, r, d = gpu.step(torch.from_numpy(acts[t]).cuda())
        o2, r2, d2 = ref.step(acts[t][sample])
        assert (o.cpu().numpy()[sample] == o2).all(), t
        assert (r.cpu().numpy()[sample] == r2).all() and (d.cpu().numpy()[sample] == d2).all()
    assert_same_state(gpu.get_state()[sample], ref.get_state(), f"{cfg} sample")


def test_sampled_parity_at_cfg2_size():
    """cfg2 at full size (4096 envs, R1, fs=4, GRAY84, default K=30) in the bench's launch
    configuration; 48 sampled envs replayed one by one in the oracle."""
    import oracle
    from paper_1907_08467_b200 import Env
    rom = games.build_rom("R1")
    N, steps = 4096, 12
    gpu = Env([rom], N, 4)
    check_engine(gpu)
    gpu.reset(0)
    acts = H.random_actions(N, steps, 1234)
    sample = np.unique(np.concatenate([np.arange(0, 16), np.arange(N - 8, N),
                                       np.random.default_rng(0).integers(0, N, 24)]))
    ref = oracle.OracleEnv([rom], len(sample), 4, H.palette_rgb())
    ref.set_env_ids(sample)
    ref.reset(0)
    for t in range(steps):
        o, r, d = gpu.step(torch.from_numpy(acts[t]).cuda())
        o2, r2, d2 = ref.step(acts[t][sample])
        assert (o.cpu().numpy()[sample] == o2).all() and (r.cpu().numpy()[sample] == r2).all()
        assert (d.cpu().numpy()[sample] == d2).all()
    assert_same_state(gpu.get_state()[sample], ref.get_state(), "cfg2 sample")


@pytest.mark.parametrize("roms", [["R1"], ["R1", "R2", "R3", "R4"]])
def test_frame_stack_parity(roms):
    """Inference path (R#32): the device frame stack
    u8[N][4][84][84] after cule_reset_stacked and every cule_step_stacked equals the oracle's,
    bit for bit, with episode ends (an 8-frame cap plus the games' own terminals) on every env."""
    import oracle
    from paper_1907_08467_b200 import Env
    rl = [games.build_rom(n) for n in roms]
    n = 70
    cfg = dict(reset_cache_size=5, max_episode_frames=8 * 4 + 4)
    gpu = Env(rl, n, 4, **cfg)
    check_engine(gpu)
    ref = oracle.OracleEnv(rl, n, 4, H.palette_rgb(), obs_mode=1, **cfg)
    stack = gpu.new_stack()
    gpu.reset_stacked(stack, 11)
    rstack = ref.reset_stacked(11)
    assert (stack.cpu().numpy() == rstack).all(), "reset stacks differ"
    acts = H.random_actions(n, 25, 99)
    n_done = 0
    for t in range(25):
        r, d = gpu.step_stacked(torch.from_numpy(acts[t]).cuda(), stack, t % 4)
        r2, d2 = ref.step_stacked(acts[t], rstack, t % 4)
        assert (r.cpu().numpy() == r2).all() and (d.cpu().numpy() == d2).all(), t
        s = stack.cpu().numpy()
        if not (s == rstack).all():
            bad = np.nonzero((s != rstack).reshape(n, -1).any(1))[0]
            raise AssertionError(f"step {t}: stacks differ for envs {bad[:8].tolist()}")
        n_done += int(d2.sum())
    assert_same_state(gpu.get_state(), ref.get_state(), "end")
    assert n_done >= n


@pytest.mark.parametrize("src", ["R1", "R2", "R4", "m20", "m21"])
def test_idle_skip_is_exact(src, engine):
    """The exact idle-loop skip (cule_config.idle_skip; R#24) skips
    whole [timer read; branch back] poll iterations in closed form: observations, rewards,
    dones, counters and the full state stay bit-identical to the oracle, which never skips."""
    if engine in ("jit", "vjit", "wsvjit"):
        pytest.skip("the translated engines have no idle-loop skip (cule_create rejects the combination)")
    import oracle
    from paper_1907_08467_b200 import Env
    rom = games.build_rom(src) if src.startswith("R") else micro.build(
        micro.m20_timer_polls() if src == "m20" else micro.m21_timint_spin(100))
    roms = [rom, games.build_rom("R1")]
    n = 40
    gpu = Env(roms, n, 4, reset_cache_size=4, idle_skip=1)
    check_engine(gpu)
    ref = oracle.OracleEnv(roms, n, 4, H.palette_rgb(), reset_cache_size=4)
    run_parity(gpu, ref, 30, seed=77)


# ---- delayed register effects (opt-in; R#35) -----------------
def _delay_programs():
    # mid-line PF1 and GRP0 writes at every residue of the playfield cell (x = 6k - 26 on row 0;
    # tests/test_oracle_delays.py pins the frames), plus a collision read of the result
    out = []
    for k in (8, 10, 12):
        row0 = "    NOP\n" * k + "    LDA #$FF\n    STA $0E\n" + "    NOP\n" * 2 + "    LDA #$00\n    STA $1B\n"
        out.append(micro.static_frame(pokes=[(0x09, 0x1E), (0x08, 0x44), (0x06, 0x86), (0x1B, 0xFF), (0x0E, 0x00)],
                                      positions=[(0x10, 16)], kernel_row0=row0, store_collisions=True))
    # mid-line RESP0 / RESM1 (RESxx start delay, R#36) with copies, a missile and a playfield to
    # collide with; the reset at the end of row 0 leaves the delay pending into the frame's end
    for k, nusiz in ((10, 3), (14, 0x16), (30, 1)):
        row0 = ("    NOP\n" * k + "    STA $10\n    STA $13\n")
        out.append(micro.static_frame(pokes=[(0x09, 0x1E), (0x06, 0x86), (0x07, 0xC8), (0x1B, 0xFF), (0x04, nusiz),
                                             (0x05, nusiz), (0x1E, 2), (0x0D, 0xF0)],
                                      positions=[(0x10, 10), (0x13, 12)], kernel_row0=row0, store_collisions=True))
    # a frame that ends (VSYNC) on the line of a visible RESP0: the start delay is pending at the
    # frame boundary (snapshot byte 63) and shows on the next frame's line 0 (window at ystart 0)
    out.append(micro.m23_resp_at_vsync())
    # HMCLR right after a visible RESP0 on the same line: the start delay stays (R#36 is cleared
    # only by the line end; HMCLR zeroes the motion registers alone), so the first copy stays dark
    row0 = "    NOP\n" * 10 + "    STA $10\n    STA $2B\n"
    out.append(micro.static_frame(pokes=[(0x09, 0x1E), (0x06, 0x86), (0x1B, 0xFF), (0x04, 0), (0x0D, 0xF0)],
                                  positions=[(0x10, 10)], kernel_row0=row0, store_collisions=True))
    return out


@pytest.mark.parametrize("case", range(8))
def test_tia_delays_static_frames_raw(case):
    """Static frames with mid-line playfield, GRP and RESxx writes, RAW frames every step, with
    the delayed register effects on (R#35, R#36): frames, collision latches and the state
    (byte 63 included) equal the oracle's."""
    rom = micro.build(_delay_programs()[case])
    gpu, ref = pair([rom], 8, 1, "raw", reset_cache_size=2, startup_frames=4, max_random_frames=3,
                    tia_delays=1, ystart=0 if case == 6 else 34)
    run_parity(gpu, ref, 6)


def test_tia_delays_games_gray84():
    """The four game ROMs (mid-line PF and GRP writes every line) with the delays on."""
    roms = [games.build_rom(n) for n in ("R1", "R2", "R3", "R4")]
    gpu, ref = pair(roms, 70, 4, reset_cache_size=4, tia_delays=1)
    run_parity(gpu, ref, 16, check_every=5)
