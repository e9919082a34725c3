python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/gpu_tests.log
for l in 32 16 8 4; do
  PADSIM_J_LPW=$l python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench24_cfg3_l$l.log 2>&1
done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench24_cfg4.log 2>&1
tail -4 gpurun_out/gpu_tests.log
