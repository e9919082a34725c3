python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/gpu_tests.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench25_cfg4.log 2>&1
python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench25_cfg2.log 2>&1
python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench25_cfg3.log 2>&1
tail -4 gpurun_out/gpu_tests.log
