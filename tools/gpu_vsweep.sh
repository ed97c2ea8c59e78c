#!/bin/bash
# VJIT engine: envs-per-warp x env-count sweep on R1 (cfg2 ROM) and the cfg4 mix, then ncu --set full
# captures of cule_vjit_step at cfg4 (32 envs/warp) and cfg3 (16 envs/warp).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
: > gpurun_out/vsweep.txt
for c in cfg2 cfg4; do
for n in ${NS:-4096 8192 16384 32768 65536}; do
for v in ${VEPWS:-8 16 32}; do
CULE_ENGINE=vjit CULE_VEPW=$v timeout 300 python bench.py --config $c --envs $n --steps 20 --warmup 10 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 1 > gpurun_out/vs.json 2> gpurun_out/vs.err
python -c "import json; d=json.loads(open('gpurun_out/vs.json').read().strip().splitlines()[-1]); print('$c', $n, 'vepw', $v, round(d['value']), round(d['ms_per_step'],3), d['config']['engine'])" >> gpurun_out/vsweep.txt 2>&1 || echo "$c $n $v FAILED" >> gpurun_out/vsweep.txt
done; done; done
cat gpurun_out/vsweep.txt
if [ -z "$NONCU" ]; then
CULE_ENGINE=vjit CULE_VEPW=32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_vjit_step -s 12 -c 1 -o gpurun_out/prof_v_cfg4 python bench.py --config cfg4 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_v_cfg4.log 2>&1; echo "ncu v cfg4 rc=$?"
CULE_ENGINE=vjit CULE_VEPW=16 timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_vjit_step -s 12 -c 1 -o gpurun_out/prof_v_cfg3 python bench.py --config cfg3 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_v_cfg3.log 2>&1; echo "ncu v cfg3 rc=$?"
fi
