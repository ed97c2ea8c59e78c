#!/bin/bash
# Engine crossover sweep (scalar vs batched SIMT) on cfg2/cfg3/cfg4, and ncu captures of the
# default engine's step kernel on cfg3/cfg4 (per-frame warp-instruction constants).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in cfg2 cfg3 cfg4; do
  for eng in scalar simt; do
    CULE_ENGINE=$eng timeout 600 python bench.py --config $cfg --steps 60 --warmup 10 --no-cpu-baseline --no-variant --e2e-steps 2 --inference-steps 0 --vtrace 0 > gpurun_out/e_${cfg}_${eng}.json 2>gpurun_out/e_${cfg}_${eng}.err
    python -c "import json; d=json.loads(open('gpurun_out/e_${cfg}_${eng}.json').read().strip().splitlines()[-1]); print('$cfg $eng', round(d['value']), round(d['ms_per_step'],3))" || tail -3 gpurun_out/e_${cfg}_${eng}.err
  done
done
if [ -n "$NCU" ]; then
for cfg in cfg3 cfg4; do
  timeout 900 ncu --set full --clock-control none -k regex:"scalar_kernel|step_kernel" -s 3 -c 1 -o gpurun_out/prof_$cfg python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 > gpurun_out/ncu_$cfg.log 2>&1; echo "ncu $cfg rc=$?"
done
fi
