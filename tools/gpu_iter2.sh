#!/bin/bash
# iteration: GPU parity (all engines), bench cfg2/cfg3/cfg4 (AUTO engines), ncu of the cfg2 and cfg4 step kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout ${PT:-1800} python -m pytest ${TESTS:-tests/test_gpu_parity.py} -q -m gpu -x ${KARG} > gpurun_out/pytest_it.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_it.log
for c in ${CFGS:-cfg2 cfg3 cfg4}; do
timeout 600 python bench.py --config $c --steps ${STEPS:-60} --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > gpurun_out/bi_${c}.json 2> gpurun_out/bi_${c}.err
python -c "import json; d=json.loads(open('gpurun_out/bi_${c}.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -5 gpurun_out/bi_${c}.err
done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_v?jit_step -s 25 -c 1 -o gpurun_out/prof_i_cfg2 python bench.py --config cfg2 --steps 3 --warmup 25 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_i_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_v?jit_step -s 12 -c 1 -o gpurun_out/prof_i_cfg4 python bench.py --config cfg4 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_i_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
fi
