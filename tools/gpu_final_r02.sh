#!/bin/bash
# Round-2 evidence: build + smoke, every GPU test, the default bench line (the driver's command), the
# reference arm, cfg3/cfg4/cfg5 lines, the ncu launch list of the bench command and ncu --set full
# captures of the step kernels (cfg2 JIT, cfg3 and cfg4 VJIT).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
if [ -z "$NOTESTS" ]; then
timeout ${PT:-3300} python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1]); print('bench', round(d['value']), d['ms_per_step'], d['config']['engine'], round(d['e2e']['value']), round(d['inference']['value']), d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 150 gpurun_out/bench_ref.json
for c in cfg3 cfg4 cfg5; do
timeout 900 python bench.py --config $c --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 10 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
python -c "import json; d=json.loads(open('gpurun_out/b_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), d['ms_per_step'], d['config']['engine'], round(d['e2e']['value']))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_v?jit -s 250 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 3 --warmup 250 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu cfg2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_v?jit -s 250 -c 1 -o gpurun_out/prof_cfg3 python bench.py --config cfg3 --steps 3 --warmup 250 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_cfg3.log 2>&1; echo "ncu cfg3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_v?jit -s 250 -c 1 -o gpurun_out/prof_cfg4 python bench.py --config cfg4 --steps 3 --warmup 250 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
