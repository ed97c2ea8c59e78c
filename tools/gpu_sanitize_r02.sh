#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the translated engines (JIT, VJIT, WSVJIT),
# default and with the delayed register effects, small shapes.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
cat > gpurun_out/san.py <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_1907_08467_b200 import Env
from paper_1907_08467_b200.inputs import games
engine = sys.argv[1]
os.environ["CULE_ENGINE"] = engine
for delays in (0, 1):
    for mode in ("gray84", "raw"):
        env = Env([games.build_rom("R3"), games.build_rom("R2")], 40, 4, obs_mode=mode, reset_cache_size=2,
                  max_random_frames=1, tia_delays=delays, max_episode_frames=12)
        assert env.engine == engine, env.engine
        env.reset(0)
        for t in range(4):
            env.step(torch.randint(0, 18, (40,), dtype=torch.uint8, device="cuda"))
        if mode == "gray84":
            st = env.new_stack()
            env.reset_stacked(st, 1)
            for t in range(3):
                env.step_stacked(torch.randint(0, 18, (40,), dtype=torch.uint8, device="cuda"), st, t % 4)
        torch.cuda.synchronize()
        env.close()
print("san ok", engine)
PY
: > gpurun_out/sanitizer_r02.txt
for e in jit vjit wsvjit; do
for tool in memcheck racecheck synccheck; do
echo "== $e $tool" >> gpurun_out/sanitizer_r02.txt
timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python gpurun_out/san.py $e >> gpurun_out/sanitizer_r02.txt 2>&1; echo "$e $tool rc=$?"
tail -2 gpurun_out/sanitizer_r02.txt
done; done
