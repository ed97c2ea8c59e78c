#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/build_old.log 2>&1)
for rep in 1 2; do
for t in new old; do
if [ $t = old ]; then d=ab_old; else d=.; fi
(cd $d && timeout 600 python bench.py --config cfg2 --steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > /tmp/ab_$t.json 2> /tmp/ab_$t.err)
python -c "import json; d=json.loads(open('/tmp/ab_$t.json').read().strip().splitlines()[-1]); print('rep $rep $t cfg2', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -3 /tmp/ab_$t.err
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tia_delays or wsvjit or (jit and not vjit)" > gpurun_out/pytest_ab2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab2.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python gpurun_out/san.py wsvjit > gpurun_out/san_ws_sync.txt 2>&1; echo "ws synccheck rc=$?"; tail -2 gpurun_out/san_ws_sync.txt
