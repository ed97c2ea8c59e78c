#!/bin/bash
# EXPERIMENT (timing only, outputs invalid): step kernel with all TIA work removed, to bound
# what a CPU-only kernel with a small register budget could reach.  Restores the sources after.
cp paper_1907_08467_b200/csrc/cpu.cuh /tmp/cpu.bak; cp paper_1907_08467_b200/csrc/kernels.cuh /tmp/kernels.bak
python tools/experiments/patch_no_tia.py
for mb in 1 6; do
  CULE_NVCC_EXTRA="-DCULE_EXP_NO_TIA -DCULE_MINB=$mb" python -c "from paper_1907_08467_b200 import build; build.build(force=True)"
  for e in 1 2 4 8; do
    echo -n "NO_TIA MINB=$mb EPW=$e "; CULE_EPW=$e python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | cut -c1-90
  done
done
cp /tmp/cpu.bak paper_1907_08467_b200/csrc/cpu.cuh; cp /tmp/kernels.bak paper_1907_08467_b200/csrc/kernels.cuh
