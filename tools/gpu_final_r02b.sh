#!/bin/bash
# final evidence (tools/gpu_final_r02.sh) + the JIT/VJIT crossover at 8192 envs after the VJIT write elision
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
bash tools/gpu_final_r02.sh
for c in cfg2 cfg4; do for e in jit vjit; do
CULE_ENGINE=$e timeout 300 python bench.py --config $c --envs 8192 --steps 30 --warmup 10 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 1 > /tmp/s.json 2>/tmp/s.err
python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print('xover $c 8192 $e', round(d['value']), round(d['ms_per_step'],3))" || echo "xover $c $e FAILED"
done; done
