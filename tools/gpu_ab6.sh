#!/bin/bash
# same-box A/B (current tree vs ab_old/ = HEAD) at cfg2 (JIT), 3 repetitions each; ncu of the new cfg2 kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/build_old.log 2>&1); echo "build old rc=$?"
for c in ${CFGS:-cfg2}; do for rep in 1 2 3; do for t in new old; do
if [ $t = old ]; then d=ab_old; else d=.; fi
(cd $d && timeout 600 python bench.py --config $c --steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --inference-steps 0 --vtrace 0 --e2e-steps 2 > /tmp/ab_$t.json 2> /tmp/ab_$t.err)
python -c "import json; d=json.loads(open('/tmp/ab_$t.json').read().strip().splitlines()[-1]); print('rep $rep $t $c', round(d['value']), d['ms_per_step'], d['config']['engine'])" || tail -3 /tmp/ab_$t.err
done; done; done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cule_v?jit_step -s 25 -c 1 -o gpurun_out/prof_ab6_cfg2 python bench.py --config cfg2 --steps 3 --warmup 25 --no-cpu-baseline --no-variant --e2e-steps 1 --inference-steps 0 --vtrace 0 --sweep 0 --e4 0 > gpurun_out/ncu_ab6_cfg2.log 2>&1; echo "ncu cfg2 rc=$?"
fi
