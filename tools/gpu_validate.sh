#!/bin/bash
# One-shot validation on a GPU box: smoke, full-size parity, torchrun path, compute-sanitizer.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size or cfg2_size" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "mapper and scalar" 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | cut -c1-200
cat > /tmp/san.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1907_08467_b200 import Env
from paper_1907_08467_b200.inputs import games
from paper_1907_08467_b200.vtrace import vtrace
for engine in ("scalar", "simt"):
    os.environ["CULE_ENGINE"] = engine
    for mode in ("gray84", "raw"):
        env = Env([games.build_rom("R3"), games.build_rom("R2")], 40, 4, obs_mode=mode, reset_cache_size=2, max_random_frames=1)
        env.reset(0)
        for t in range(3):
            env.step(torch.randint(0, 18, (40,), dtype=torch.uint8, device="cuda"))
        if mode == "gray84":  # frame stack path, with episode ends
            st = env.new_stack()
            env.reset_stacked(st, 1)
            for t in range(4):
                env.step_stacked(torch.randint(0, 18, (40,), dtype=torch.uint8, device="cuda"), st, t % 4)
        env.debug_exec(50)
        torch.cuda.synchronize()
        env.close()
r = torch.randn(20, 333, device="cuda")
vtrace(r, r.clone(), torch.randn(333, device="cuda"), r * 0.1, r * 0.2, (r > 1).to(torch.uint8), 0.99)
torch.cuda.synchronize()
print("sanitizer workload done")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python /tmp/san.py > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.txt
done
