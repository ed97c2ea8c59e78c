set -x
python -m pytest tests/test_gpu_parity.py -q -m gpu -k "scalar" -x 2>&1 | tail -3 > gpurun_out/t_s.log
CULE_ENGINE=scalar timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/b_s.log 2>&1
CULE_ENGINE=scalar timeout 300 ncu --set full --clock-control none --import-source on -k regex:scalar_kernel -s 2 -c 1 -o gpurun_out/prof_s python bench.py --steps 2 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_s.log 2>&1
