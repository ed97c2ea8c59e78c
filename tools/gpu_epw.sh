#!/bin/bash
# VJIT envs per warp at 16384 envs after the write elision: cfg3 (R2) and R1 / the cfg4 mix at 16384
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
B="--steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2"
for rep in 1 2; do for cfgn in "cfg3" "cfg2 --envs 16384" "cfg4 --envs 16384"; do for v in 8 16 32; do
CULE_ENGINE=vjit CULE_VEPW=$v timeout 600 python bench.py --config $cfgn $B > /tmp/e.json 2> /tmp/e.err
python -c "import json; d=json.loads(open('/tmp/e.json').read().strip().splitlines()[-1]); print('rep $rep', '$cfgn', 'epw $v', round(d['value']), round(d['ms_per_step'],3))" || tail -2 /tmp/e.err
done; done; done
