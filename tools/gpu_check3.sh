#!/bin/bash
# delays parity on every engine + vjit/simt parity after the mask cache; mask-cache A/B at cfg3/cfg4; cfg2 line
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tia_delays or (vjit and not wsvjit) or simt" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c3.log
for c in cfg4 cfg3; do for nc in 0 1; do
if [ $nc = 1 ]; then export CULE_TIA_NO_MASK_CACHE=1; else unset CULE_TIA_NO_MASK_CACHE; fi
timeout 600 python bench.py --config $c --steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > gpurun_out/bm_${c}_$nc.json 2> gpurun_out/bm_${c}_$nc.err
python -c "import json; d=json.loads(open('gpurun_out/bm_${c}_$nc.json').read().strip().splitlines()[-1]); print('$c nocache=$nc', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -3 gpurun_out/bm_${c}_$nc.err
done; done
unset CULE_TIA_NO_MASK_CACHE
timeout 600 python bench.py --config cfg2 --steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > gpurun_out/bm_cfg2.json 2> gpurun_out/bm_cfg2.err
python -c "import json; d=json.loads(open('gpurun_out/bm_cfg2.json').read().strip().splitlines()[-1]); print('cfg2', round(d['value']), d['ms_per_step'], d['config']['engine'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_vjit -s 12 -c 1 -o gpurun_out/prof_c3_cfg4 python bench.py --config cfg4 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"
