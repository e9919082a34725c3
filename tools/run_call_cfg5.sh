mkdir -p gpurun_out/cfg5
timeout 2400 python bench.py --config cfg5 --steps 1 --warmup 3 --e2e-steps 1 --cpu-seconds 20 > gpurun_out/cfg5/bench_cfg5.log 2>&1
tail -2 gpurun_out/cfg5/bench_cfg5.log
