#!/bin/bash
# VJIT engine iteration: parity tests on the vjit engine, then bench lines, then (optional) ncu.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout ${PT:-900} python -m pytest ${TESTS:-tests/test_gpu_parity.py} -q -m gpu -x -k "vjit ${KSEL}" > gpurun_out/pytest_vjit.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_vjit.log
for c in ${CFGS:-cfg4 cfg3}; do
CULE_ENGINE=vjit timeout 600 python bench.py --config $c --steps 30 --warmup 10 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > gpurun_out/bv_${c}.json 2> gpurun_out/bv_${c}.err
python -c "import json; d=json.loads(open('gpurun_out/bv_${c}.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -5 gpurun_out/bv_${c}.err
done
if [ -n "$NCU" ]; then
CULE_ENGINE=vjit timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_vjit_step -s 12 -c 1 -o gpurun_out/prof_v_cfg4 python bench.py --config cfg4 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_v_cfg4.log 2>&1; echo "ncu v cfg4 rc=$?"
fi
