#!/bin/bash
# engine crossover after the i-cache fix: VJIT (envs per warp 4..32) vs JIT at 4096-32768 envs, R1 and the cfg4 mix;
# NEXT-2 ablation re-run (VJIT vs WSVJIT at cfg3/cfg4)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/sweep2.txt
for c in cfg2 cfg4; do for n in 4096 8192 16384 32768; do
CULE_ENGINE=jit timeout 300 python bench.py --config $c --envs $n --steps 30 --warmup 10 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 1 > /tmp/s.json 2>/tmp/s.err
python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print('$c', $n, 'jit', '-', round(d['value']), round(d['ms_per_step'],3))" >> gpurun_out/sweep2.txt 2>&1 || echo "$c $n jit FAILED" >> gpurun_out/sweep2.txt
for v in 4 8 16 32; do
CULE_ENGINE=vjit CULE_VEPW=$v timeout 300 python bench.py --config $c --envs $n --steps 30 --warmup 10 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 1 > /tmp/s.json 2>/tmp/s.err
python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print('$c', $n, 'vjit', $v, round(d['value']), round(d['ms_per_step'],3))" >> gpurun_out/sweep2.txt 2>&1 || echo "$c $n vjit $v FAILED" >> gpurun_out/sweep2.txt
done; done; done
cat gpurun_out/sweep2.txt
for c in cfg4 cfg3; do for e in vjit wsvjit; do
CULE_ENGINE=$e timeout 600 python bench.py --config $c --steps 60 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > gpurun_out/bw_${c}_$e.json 2> gpurun_out/bw_${c}_$e.err
python -c "import json; d=json.loads(open('gpurun_out/bw_${c}_$e.json').read().strip().splitlines()[-1]); print('$c', '$e', round(d['value']), 'FPS', round(d['ms_per_step'],3), 'ms/step')"
done; done
