#!/bin/bash
# VJIT engine iteration: parity tests on the vjit engine, then cfg3/cfg4 bench lines per envs-per-warp.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout ${PT:-900} python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vjit ${KSEL}" > gpurun_out/pytest_vjit.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_vjit.log
for c in ${CFGS:-cfg4 cfg3 cfg2}; do
for v in ${VEPWS:-32 16}; do
CULE_ENGINE=vjit CULE_VEPW=$v timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > gpurun_out/bv_${c}_$v.json 2> gpurun_out/bv_${c}_$v.err
python -c "import json; d=json.loads(open('gpurun_out/bv_${c}_$v.json').read().strip().splitlines()[-1]); print('$c vepw $v', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -5 gpurun_out/bv_${c}_$v.err
done
done
