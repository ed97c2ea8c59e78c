#!/bin/bash
# parity (per-lane engines + delays) after the dp4a epilogue / log capacity 64; log-capacity A/B at cfg3/cfg4; ncu cfg4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vjit or simt or tia_delays" > gpurun_out/pytest_it4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_it4.log
for c in cfg4 cfg3; do for cap in 64 32; do
CULE_VLOGCAP=$cap timeout 600 python bench.py --config $c --steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > /tmp/b.json 2> /tmp/b.err
python -c "import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$c logcap $cap', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -3 /tmp/b.err
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_vjit -s 12 -c 1 -o gpurun_out/prof_it4_cfg4 python bench.py --config cfg4 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_it4.log 2>&1; echo "ncu rc=$?"
