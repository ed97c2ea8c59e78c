"""Pins for the oracle's step / reset-cache / preprocessing layer (SURVEY.md §8(c).10-12,
§8(c).14 rows 14-15, 17, 20-23)."""
import os

import numpy as np
import pytest

import helpers as H
from paper_1907_08467_b200.inputs import games, micro

GOLDEN_AREA = os.path.join(os.path.dirname(__file__), "golden", "area84_weights.txt")


# ---------------------------------------------------------------------------------------------
# preprocessing
# ---------------------------------------------------------------------------------------------
def golden_weights():
    rows, cols = {}, {}
    for ln in open(GOLDEN_AREA):
        if ln.startswith("#") or not ln.strip():
            continue
        head, rest = ln.split(":", 1)
        kind, idx = head.split()
        pairs = [tuple(int(v) for v in p.split(":")) for p in rest.split()]
        (rows if kind == "rows" else cols)[int(idx)] = pairs
    WR = np.zeros((84, 210), np.int64)
    for i in range(84):
        m, par = divmod(i, 2)
        for off, w in rows[par]:
            WR[i, 5 * m + off] = w
    WC = np.zeros((84, 160), np.int64)
    for j in range(84):
        q, t = divmod(j, 21)
        for off, w in cols[t]:
            WC[j, 40 * q + off] = w
    return WR, WC


def area84_from_table(img):
    WR, WC = golden_weights()
    S = WR @ img.astype(np.int64) @ WC.T
    q, r = S // 200, S % 200
    return (q + ((r > 100) | ((r == 100) & (q & 1 == 1)))).astype(np.uint8)


def test_golden_weights_sum():
    WR, WC = golden_weights()
    assert (WR.sum(1) == 5).all() and (WC.sum(1) == 40).all()
    assert (WR.sum(0) == 2).all() and (WC.sum(0) == 21).all()   # every input fully covered


def test_area84_matches_golden_table(orc):
    rng = np.random.default_rng(3)
    for _ in range(20):
        img = rng.integers(0, 256, (210, 160), dtype=np.uint8)
        assert (orc.area84(img) == area84_from_table(img)).all()
    for v in (0, 1, 77, 128, 255):   # uniform frames are exact
        assert (orc.area84(np.full((210, 160), v, np.uint8)) == v).all()


def test_area84_vs_cv2_inter_area(orc):
    cv2 = pytest.importorskip("cv2")
    rng = np.random.default_rng(4)
    mism = 0
    for _ in range(10):
        img = rng.integers(0, 256, (210, 160), dtype=np.uint8)
        ref = cv2.resize(img, (84, 84), interpolation=cv2.INTER_AREA).astype(np.int32)
        got = orc.area84(img).astype(np.int32)
        assert np.abs(ref - got).max() <= 1      # S:338 +-1 vs an area oracle
        mism += int((ref != got).sum())
    assert mism / (10 * 84 * 84) < 0.01          # differences only at exact ties [R#17]


def test_gray_lut(orc):
    g = orc.gray_lut(H.palette_rgb())
    rgb = np.frombuffer(H.palette_rgb(), np.uint8).reshape(128, 3)
    gray_rows = (rgb[:, 0] == rgb[:, 1]) & (rgb[:, 1] == rgb[:, 2])
    assert gray_rows.sum() >= 8
    assert (g[gray_rows] == rgb[gray_rows, 0]).all()   # R=G=B=v -> v (weights sum to 1000)
    assert g[0] == 0                                   # black stays black


def test_splitmix64_reference_vectors(orc):
    # canonical SplitMix64 outputs for state 0: first two values of the published generator
    L = orc.lib()
    assert L.orc_splitmix64(0) == 0xE220A8397B1DCDAF
    assert L.orc_splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


# ---------------------------------------------------------------------------------------------
# env layer
# ---------------------------------------------------------------------------------------------
R1 = games.build_rom("R1")


def make_env(orc, roms=(R1,), n=4, fs=4, **cfg):
    cfg.setdefault("reset_cache_size", 4)
    return orc.OracleEnv(list(roms), n, fs, H.palette_rgb(), **cfg)


def test_create_validation(orc):
    with pytest.raises(ValueError, match="-2"):
        make_env(orc, roms=(bytes(5000),))           # S:182 UnsupportedRomSize
    with pytest.raises(ValueError, match="-1"):
        make_env(orc, fs=0)
    with pytest.raises(ValueError, match="-3"):
        make_env(orc, roms=(micro.build(micro.m14_jam(3)),))   # JAM during the cache build


def test_cache_k1_and_r0(orc):
    e = make_env(orc, n=6, reset_cache_size=1)
    e.reset(0)
    st = e.get_state()
    for i in range(1, 6):   # S:272 K=1 -> every env holds the single entry
        assert (st[i, H.MACHINE_BYTES] == st[0, H.MACHINE_BYTES]).all()
    e = make_env(orc, reset_cache_size=5, max_random_frames=0)
    cs, co = e.cache()
    for k in range(1, 5):   # S:253 R=0 -> identical entries
        assert (cs[k] == cs[0]).all() and (co[k] == co[0]).all()


def test_cache_seed_determinism_and_provenance(orc):
    a = make_env(orc, n=8, seed=11)
    b = make_env(orc, n=8, seed=11)
    c = make_env(orc, n=8, seed=12)
    ca, cb, cc = a.cache()[0], b.cache()[0], c.cache()[0]
    assert (ca == cb).all()
    assert not (ca == cc).all()
    oa = a.reset(5)
    ob = b.reset(5)
    assert (oa == ob).all() and (a.get_state() == b.get_state()).all()
    acts = H.random_actions(8, 60)
    for t in range(60):
        ra = a.step(acts[t])
        rb = b.step(acts[t])
        for x, y in zip(ra, rb):
            assert (x == y).all()
        st = a.get_state()
        for i in range(8):
            if ra[2][i]:   # S:270 provenance: machine part equals a cache entry
                assert any((st[i, H.MACHINE_BYTES] == ca[k, H.MACHINE_BYTES]).all()
                           for k in range(len(ca)))
                assert H.episode_frames(st[i]) == 0 and H.episode_return(st[i]) == 0


def _splitmix(x):
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def _H(a, b):
    return _splitmix(a ^ _splitmix(b))


def test_reset_picks_and_cache_lengths(orc):
    K, R, seed = 6, 30, 3
    e = make_env(orc, n=10, reset_cache_size=K, seed=seed, obs_mode=0)
    cs, co = e.cache()
    obs = e.reset(99)
    st = e.get_state()
    for g in range(10):
        k = _H(_H(99, g), 0) % K                 # pick(seed, g, 0) [R#22]
        assert (st[g, H.MACHINE_BYTES] == cs[k, H.MACHINE_BYTES]).all()
        assert (obs[g] == co[k]).all()
        bcd = lambda b: 10 * (b >> 4) + (b & 15)
        score = 100 * bcd(H.ram(st[g], 0x80)) + bcd(H.ram(st[g], 0x81))
        assert H.episode_index(st[g]) == 0 and H.prev_score(st[g]) == score
    # entry k ran 64 + u_k frames; frames differ in length only through u_k, so entries with
    # equal u_k are identical
    us = [_H(seed ^ 0x5245534554434143, k) % (R + 1) for k in range(K)]
    for i in range(K):
        for j in range(K):
            if us[i] == us[j]:
                assert (cs[i] == cs[j]).all()


def test_m17_reward_and_done(orc):
    rom = micro.build(micro.m17_score())
    e = make_env(orc, roms=(rom,), n=2, fs=4)
    e.reset(0)
    total = 0
    done_step = None
    for t in range(45):
        _, rew, done = e.step(np.array([1, 0], np.uint8))   # env 0 holds FIRE, env 1 NOOP
        assert rew[1] == 0 and done[1] == 0
        total += int(rew[0])
        if done[0]:
            done_step = t
            break
        assert rew[0] == 4                                  # BCD score +1 per frame, fs = 4
    # score crosses 99 -> 100 (BCD carry) and reaches 150 in frame 150 -> done at step 37
    assert done_step == 37 and total == 152
    c = e.counters()
    assert c[1] == 1 and c[2] == 152 and c[3] == 0 and c[0] == 2 * 4 * 38


@pytest.mark.parametrize("src", [micro.m14_jam(120), micro.m15_no_vsync(120)])
def test_faults_isolated(orc, src):
    rom = micro.build(src)
    e = make_env(orc, roms=(rom, R1), n=4, fs=4, reset_cache_size=2, max_random_frames=0,
                 obs_mode=0)
    e.reset(0)
    saw = False
    for t in range(20):
        obs, rew, done = e.step(np.zeros(4, np.uint8))
        assert not done[1] and not done[3]                  # R1 envs unaffected
        if done[0]:
            saw = True
            assert rew[0] == 0 and (obs[0] == 0).all()       # fault: reward 0, zero obs
            assert e.counters()[3] >= 1
            st = e.get_state()
            assert st[0, H.OFF["fault"]] == 0 and H.episode_index(st[0]) == 1
            break
    assert saw


def test_render_purity_raw_vs_gray(orc):
    # rendering never changes machine state, reward or done
    acts = H.random_actions(4, 40, seed=5)
    a = make_env(orc, obs_mode=0)
    b = make_env(orc, obs_mode=1)
    a.reset(1)
    b.reset(1)
    for t in range(40):
        _, ra, da = a.step(acts[t])
        _, rb, db = b.step(acts[t])
        assert (ra == rb).all() and (da == db).all()
        assert (a.get_state() == b.get_state()).all()


def test_gray84_obs_composition(orc):
    # GRAY84 obs = area84(max(gray(frame fs-1), gray(frame fs))) of the frames RAW mode renders
    gray = H.gray_of_palette()
    acts = H.random_actions(2, 12, seed=9)
    raw = make_env(orc, n=2, fs=1, obs_mode=0)
    g2 = make_env(orc, n=2, fs=2, obs_mode=1)
    raw.reset(2)
    g2.reset(2)
    for t in range(12):
        oA, _, dA = raw.step(acts[t])
        oB, _, dB = raw.step(acts[t])
        og, _, dg = g2.step(acts[t])
        if dA.any() or dB.any() or dg.any():
            break
        for i in range(2):
            m = np.maximum(gray[oA[i]], gray[oB[i]])
            assert (og[i] == area84_from_table(m)).all()


def test_frameskip_invariance(orc):
    # fs=4 with action a == fs=1 with a repeated 4x, at common frame counts, up to the first done
    acts = H.random_actions(3, 30, seed=8)
    e4 = make_env(orc, n=3, fs=4)
    e1 = make_env(orc, n=3, fs=1)
    e4.reset(4)
    e1.reset(4)
    for t in range(30):
        _, r4, d4 = e4.step(acts[t])
        rs = 0
        for _ in range(4):
            _, r1, d1 = e1.step(acts[t])
            rs = rs + r1
            if d1.any():
                break
        if d1.any() or d4.any():
            break
        assert (r4 == rs).all()
        s4, s1 = e4.get_state(), e1.get_state()
        assert (s4[:, H.MACHINE_BYTES] == s1[:, H.MACHINE_BYTES]).all()


def test_batched_equals_isolated_and_num_envs_independence(orc):
    # env g's trajectory depends only on (ROM, seed, g, its actions)
    roms = [games.build_rom("R1"), games.build_rom("R3")]
    acts = H.random_actions(6, 25, seed=2)
    big = make_env(orc, roms=roms, n=6)
    big.reset(7)
    outs = [big.step(acts[t]) for t in range(25)]
    for g in (0, 3, 5):
        one = make_env(orc, roms=roms, n=1, env_index_base=g)
        one.reset(7)
        for t in range(25):
            o, r, d = one.step(acts[t, g:g + 1])
            assert (o[0] == outs[t][0][g]).all() and r[0] == outs[t][1][g] and d[0] == outs[t][2][g]
    small = make_env(orc, roms=roms, n=3)
    small.reset(7)
    for t in range(25):
        o, r, d = small.step(acts[t, :3])
        assert (o == outs[t][0][:3]).all() and (r == outs[t][1][:3]).all()


def test_episode_cap(orc):
    e = make_env(orc, n=2, fs=4, max_episode_frames=20)
    e.reset(0)
    dones = [e.step(np.zeros(2, np.uint8))[2] for _ in range(6)]
    assert [int(d[0]) for d in dones] == [0, 0, 0, 0, 1, 0]   # 20 frames = 5 steps of 4
