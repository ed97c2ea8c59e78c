"""Debug helper: find the first instruction where the GPU and the oracle diverge for one env.

Runs oracle steps to a given step, then bisects the instruction count with the kernel's debug
entry (cule_debug_exec) against oracle.exec_instr.  Test/debug tool only."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import helpers as H
import oracle
from paper_1907_08467_b200 import Env
from paper_1907_08467_b200.inputs import games

def main(rom_name="R1", n=16, fs=1, mode=0, step=9, env_i=2, K=30):
    rom = games.build_rom(rom_name)
    ref = oracle.OracleEnv([rom], n, fs, H.palette_rgb(), obs_mode=mode, reset_cache_size=K)
    ref.reset(0)
    acts = H.random_actions(n, step + 1, 1234)
    for t in range(step):
        ref.step(acts[t])
    s0 = ref.get_state()
    # latch the next action into the snapshot the way the step does
    st = s0[env_i].copy()
    o1 = oracle.OracleEnv([rom], 1, 1, H.palette_rgb(), obs_mode=0, reset_cache_size=1)
    a = int(acts[step][env_i])
    # apply input latches via one zero-instruction run_frame? use exec of 0 instr after setting bytes
    up=down=left=right=fire=0
    d = {0:"",1:"F",2:"U",3:"R",4:"L",5:"D",6:"UR",7:"UL",8:"DR",9:"DL",10:"UF",11:"RF",12:"LF",13:"DF",14:"URF",15:"ULF",16:"DRF",17:"DLF"}[a]
    sw = 0xFF & ~((0x80 if "R" in d else 0)|(0x40 if "L" in d else 0)|(0x20 if "D" in d else 0)|(0x10 if "U" in d else 0))
    st[18] = sw; st[19] = 0 if "F" in d else 0x80
    gpu = Env([rom], 1, 1, obs_mode="raw", reset_cache_size=1, startup_frames=0, max_random_frames=0)
    def run_gpu(k):
        gpu.set_state(st[None])
        stat = gpu.debug_exec(k).cpu().numpy()[0]
        return stat, gpu.get_state()[0]
    def run_orc(k):
        s = st.copy(); r, _ = oracle.exec_instr(rom, s, k); return r, s
    lo, hi = 0, 8000
    sg, g = run_gpu(hi); so, o = run_orc(hi)
    print("at", hi, "status", sg, so, "equal", (g == o).all())
    while hi - lo > 1:
        mid = (lo + hi) // 2
        sg, g = run_gpu(mid); so, o = run_orc(mid)
        if (g == o).all() and sg == so: lo = mid
        else: hi = mid
    sg, g = run_gpu(hi); so, o = run_orc(hi)
    _, prev = run_orc(lo)
    cols = np.nonzero(g != o)[0]
    pc = H.pc(prev)
    print("first divergence after instruction", hi, "pc %04x" % pc, "op", rom[pc & 0xFFF:(pc & 0xFFF) + 3].hex(),
          "fc", H.fc(prev), "line", H.fc(prev)//76)
    print("bytes", cols.tolist(), "gpu", g[cols].tolist(), "oracle", o[cols].tolist())
    print("prev state hdr", prev[:64].tolist())

if __name__ == "__main__":
    args = [int(a) if a.isdigit() else a for a in sys.argv[1:]]
    main(*args)
