mkdir -p gpurun_out/c5
timeout 2400 python bench.py --config cfg5 --steps 1 --warmup 3 --e2e-steps 1 --cpu-seconds 20 > gpurun_out/c5/bench_cfg5.log 2>&1
tail -1 gpurun_out/c5/bench_cfg5.log
