#!/bin/bash
# VJIT write elision by warp vote (R#37): same-box A/B vs ab_old/ (HEAD, VJIT keeps every write) at cfg4 / cfg3;
# CULE_VELIDE=0 (same tree, elision off); the __match_any_sync scheduler ablation (CULE_VSCHED=match); VJIT parity
# (incl. full-size cfg4) with the elision and with the match scheduler; ncu cfg4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/build_old.log 2>&1); echo "build old rc=$?"
B="--steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2"
show() { python -c "import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('$1', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -3 /tmp/ab.err; }
for c in cfg4 cfg3; do for rep in 1 2; do
timeout 600 python bench.py --config $c $B > /tmp/ab.json 2> /tmp/ab.err; show "rep $rep new $c"
(cd ab_old && timeout 600 python bench.py --config $c $B > /tmp/ab.json 2> /tmp/ab.err); show "rep $rep old $c"
done
CULE_VELIDE=0 timeout 600 python bench.py --config $c $B > /tmp/ab.json 2> /tmp/ab.err; show "new-no-elision $c"
CULE_VSCHED=match timeout 600 python bench.py --config $c $B > /tmp/ab.json 2> /tmp/ab.err; show "new-match-sched $c"
CULE_VELIDE=0 CULE_VSCHED=match timeout 600 python bench.py --config $c $B > /tmp/ab.json 2> /tmp/ab.err; show "new-no-elision-match-sched $c"
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vjit" > gpurun_out/pytest_ab7.log 2>&1; echo "pytest vjit rc=$?"; tail -1 gpurun_out/pytest_ab7.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "cfg4 and vjit" > gpurun_out/pytest_ab7_full.log 2>&1; echo "pytest full cfg4 vjit rc=$?"; tail -1 gpurun_out/pytest_ab7_full.log
CULE_VSCHED=match timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vjit and not wsvjit and (gray84 or mixed or random_instructions or episode)" > gpurun_out/pytest_ab7_match.log 2>&1; echo "pytest match rc=$?"; tail -1 gpurun_out/pytest_ab7_match.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_vjit_step -s 12 -c 1 -o gpurun_out/prof_ab7_cfg4 python bench.py --config cfg4 --steps 3 --warmup 12 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_ab7_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
