#!/bin/bash
# Iteration session: build, scalar-engine parity tests, bench cfg2 (+cfg3/cfg4 on the scalar
# engine), one ncu --set full capture of the scalar kernel on cfg2.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -x -k "${TESTK:-scalar}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for cfg in ${CFGS:-cfg2 cfg3 cfg4}; do
  CULE_ENGINE=scalar timeout 600 python bench.py --config $cfg --steps 100 --warmup 20 --no-cpu-baseline --no-variant --e2e-steps 3 > gpurun_out/b_${cfg}.json 2>gpurun_out/b_${cfg}.err
  python -c "import json; d=json.loads(open('gpurun_out/b_${cfg}.json').read().strip().splitlines()[-1]); print('$cfg', round(d['value']), round(d['ms_per_step'],3), d['clocks'])" || tail -5 gpurun_out/b_${cfg}.err
done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scalar_kernel -s 5 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-variant --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full.log
fi
