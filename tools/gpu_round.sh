#!/bin/bash
# One GPU session: build, smoke, gpu tests, default bench (full contract), reference arm, bench
# cfg2/3/4 (idle skip off/on), launch list, ncu --set full of the top kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc=$?"; tail -c 400 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
for cfg in cfg2 cfg3 cfg4; do
  for sk in 0 1; do
    timeout 600 python bench.py --config $cfg --idle-skip $sk --steps 100 --warmup 20 --no-cpu-baseline --no-variant --e2e-steps 5 > gpurun_out/b_${cfg}_s$sk.json 2>gpurun_out/b_${cfg}_s$sk.err
    python -c "import json; d=json.loads(open('gpurun_out/b_${cfg}_s$sk.json').read().strip().splitlines()[-1]); print('$cfg skip=$sk', round(d['value']), round(d['ms_per_step'],3), d['clocks'])"
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-variant --e2e-steps 1 > gpurun_out/launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scalar_kernel -s 5 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-variant --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
