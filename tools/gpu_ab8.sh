#!/bin/bash
# inference-path policy (cudnn.benchmark, channels-last, 1/255 folded into conv1) A/B vs ab_old/ (HEAD), and
# compute-sanitizer on the translated engines with the TIA write elision (tools/gpu_sanitize_r02.sh)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/build_old.log 2>&1); echo "build old rc=$?"
B="--steps 100 --warmup 20 --no-cpu-baseline --sweep 0 --e4 0 --no-variant --vtrace 0 --e2e-steps 20 --inference-steps 60"
for rep in 1 2; do
timeout 600 python bench.py $B > /tmp/ab.json 2> /tmp/ab.err
python -c "import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('rep $rep new', round(d['value']), 'inference', round(d['inference']['value']), round(d['inference']['ms_per_step'],3), 'e2e', round(d['e2e']['value']))" || tail -3 /tmp/ab.err
(cd ab_old && timeout 600 python bench.py $B > /tmp/ab.json 2> /tmp/ab.err)
python -c "import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('rep $rep old', round(d['value']), 'inference', round(d['inference']['value']), round(d['inference']['ms_per_step'],3), 'e2e', round(d['e2e']['value']))" || tail -3 /tmp/ab.err
done
# sanitizer: the san.py workload of tools/gpu_sanitize_r02.sh on the two engines with the write elision
sed -n '/^cat > gpurun_out\/san.py/,/^PY$/p' tools/gpu_sanitize_r02.sh | bash
: > gpurun_out/sanitizer_r02b.txt
for e in jit vjit; do for tool in memcheck racecheck; do
echo "== $e $tool" >> gpurun_out/sanitizer_r02b.txt
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python gpurun_out/san.py $e >> gpurun_out/sanitizer_r02b.txt 2>&1; echo "$e $tool rc=$?"
tail -2 gpurun_out/sanitizer_r02b.txt
done; done
