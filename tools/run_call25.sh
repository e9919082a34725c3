python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/gpu_tests.log
for w in 0 4 16 64; do
  PADSIM_SYNC_WIN=$w python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench20_cfg4_w$w.log 2>&1
done
for w in 0 16; do
  PADSIM_SYNC_WIN=$w python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench20_cfg3_w$w.log 2>&1
done
tail -4 gpurun_out/gpu_tests.log
