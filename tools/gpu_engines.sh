#!/bin/bash
# Engine crossover sweep (scalar vs batched SIMT) on cfg2/cfg3/cfg4 + the full GPU test suite +
# ncu captures of the scalar kernel on cfg3/cfg4 (per-frame warp-instruction constants).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for cfg in cfg2 cfg3 cfg4; do
  for eng in scalar simt; do
    CULE_ENGINE=$eng timeout 600 python bench.py --config $cfg --steps 60 --warmup 10 --no-cpu-baseline --no-variant --e2e-steps 2 > gpurun_out/e_${cfg}_${eng}.json 2>gpurun_out/e_${cfg}_${eng}.err
    python -c "import json; d=json.loads(open('gpurun_out/e_${cfg}_${eng}.json').read().strip().splitlines()[-1]); print('$cfg $eng', round(d['value']), round(d['ms_per_step'],3))" || tail -3 gpurun_out/e_${cfg}_${eng}.err
  done
done
for cfg in ${NCUCFGS:-cfg3 cfg4}; do
  CULE_ENGINE=scalar timeout 900 ncu --set full --clock-control none --import-source on -k regex:scalar_kernel -s 3 -c 1 -o gpurun_out/prof_$cfg python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-variant --e2e-steps 1 > gpurun_out/ncu_$cfg.log 2>&1; echo "ncu $cfg rc=$?"
done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
