#!/bin/bash
# WSVJIT iteration: parity on wsvjit, then VJIT vs WSVJIT bench at cfg3/cfg4 (same steps), ncu of the WS kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout ${PT:-900} python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wsvjit ${KSEL}" > gpurun_out/pytest_ws.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_ws.log
for c in cfg4 cfg3; do for e in vjit wsvjit; do
CULE_ENGINE=$e timeout 600 python bench.py --config $c --steps 60 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > gpurun_out/bw_${c}_$e.json 2> gpurun_out/bw_${c}_$e.err
python -c "import json; d=json.loads(open('gpurun_out/bw_${c}_$e.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -5 gpurun_out/bw_${c}_$e.err
done; done
if [ -n "$NCU" ]; then
CULE_ENGINE=wsvjit timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_vjit_ws_step -s 12 -c 1 -o gpurun_out/prof_ws_cfg4 python bench.py --config cfg4 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_ws_cfg4.log 2>&1; echo "ncu ws cfg4 rc=$?"
fi
