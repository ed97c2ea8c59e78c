# bench both engines on cfg2/cfg3/cfg4 (one line each: engine config value ms)
for cfg in cfg2 cfg3 cfg4; do
  for e in simt scalar; do
    CULE_ENGINE=$e timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', '$cfg', round(d['value']), round(d['ms_per_step'],2))"
  done
done
