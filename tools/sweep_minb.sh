#!/bin/bash
# experiment: register budget (CULE_MINB) x envs per warp on cfg2
for mb in 1 3 4; do
  CULE_NVCC_EXTRA="-DCULE_MINB=$mb" python -c "from paper_1907_08467_b200 import build; build.build(force=True)"
  for e in 2 4 8; do
    echo -n "MINB=$mb EPW=$e "
    CULE_EPW=$e python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | cut -c1-100
  done
done
