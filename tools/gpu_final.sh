#!/bin/bash
# Evidence session: build + smoke, full GPU tests, the default bench line (the driver's
# command), the reference arm, the idle-skip variant, the ncu launch list of the bench
# command and one ncu --set full capture of the step kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
if [ -z "$NOTESTS" ]; then
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1]); print('bench', round(d['value']), d['ms_per_step'], d['e2e']['value'], d['inference']['value'], d['roofline']['frac'], d['cpu_baseline']['value'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 200 gpurun_out/bench_ref.json
timeout 600 python bench.py --idle-skip 1 --steps 100 --warmup 20 --no-cpu-baseline --e2e-steps 5 --inference-steps 0 --vtrace 0 > gpurun_out/bench_skip.json 2>/dev/null; tail -c 300 gpurun_out/bench_skip.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 > gpurun_out/launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scalar_kernel -s 5 -c 1 -o gpurun_out/prof_cfg2 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --e2e-steps 1 --inference-steps 0 --vtrace 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
