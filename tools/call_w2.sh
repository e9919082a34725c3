D=gpurun_out/w2
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_wide.py -x -q > $D/wide_tests.log 2>&1; tail -3 $D/wide_tests.log
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 3 --e2e-steps 1 --cpu-seconds 20 > $D/bench_cfg5.log 2>&1
tail -1 $D/bench_cfg5.log | cut -c1-1500
