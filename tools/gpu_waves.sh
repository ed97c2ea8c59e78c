#!/bin/bash
# VJIT block sizing beyond one wave (65536 envs): equal waves of 7-warp blocks vs one wave of 12-warp blocks + a
# short second wave (CULE_VWPB=12 reproduces the old sizing); launch-shape / env-count parity of VJIT
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
B="--steps 60 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2"
for rep in 1 2; do for cfgn in "cfg2 --envs 65536" "cfg4 --envs 65536"; do
timeout 600 python bench.py --config $cfgn $B > /tmp/e.json 2> /tmp/e.err
python -c "import json; d=json.loads(open('/tmp/e.json').read().strip().splitlines()[-1]); print('rep $rep', '$cfgn', 'new', round(d['value']), round(d['ms_per_step'],3), d['config']['engine'])" || tail -2 /tmp/e.err
CULE_VWPB=12 timeout 600 python bench.py --config $cfgn $B > /tmp/e.json 2> /tmp/e.err
python -c "import json; d=json.loads(open('/tmp/e.json').read().strip().splitlines()[-1]); print('rep $rep', '$cfgn', 'old (12 warps/block)', round(d['value']), round(d['ms_per_step'],3), d['config']['engine'])" || tail -2 /tmp/e.err
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vjit and (launch_shape or num_envs or mixed)" > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_w.log
