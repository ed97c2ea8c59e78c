#!/bin/bash
# experiment: TIA write-log capacity (entries per env) on cfg2 / cfg4
for cap in 32 64 96; do
  sed -i "s/constexpr int kLogCap = [0-9]*;/constexpr int kLogCap = $cap;/" paper_1907_08467_b200/csrc/tia.cuh
  python -c "from paper_1907_08467_b200 import build; build.build(force=True)"
  echo -n "cap=$cap cfg2 "; python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | cut -c1-100
  echo -n "cap=$cap cfg4 "; python bench.py --steps 8 --warmup 2 --no-cpu-baseline --e2e-steps 1 --config cfg4 2>&1 | tail -1 | cut -c1-100
done
