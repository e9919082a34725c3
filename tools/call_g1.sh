D=gpurun_out/g1
mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q > $D/gpu_tests.log 2>&1
tail -30 $D/gpu_tests.log
timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $D/bench_cfg3.log 2>&1
timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $D/bench_cfg4.log 2>&1
tail -2 $D/bench_cfg3.log | cut -c1-400
tail -2 $D/bench_cfg4.log | cut -c1-400
