# Full round evidence on one box: usage: bash tools/run_round.sh <tag>
tag=$1
mkdir -p gpurun_out/$tag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$tag/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/$tag/gpu_tests.log
tail -3 gpurun_out/$tag/gpu_tests.log
timeout 900 python bench.py > gpurun_out/$tag/bench_cfg4.log 2>&1; tail -1 gpurun_out/$tag/bench_cfg4.log
timeout 600 python bench.py --config cfg2 > gpurun_out/$tag/bench_cfg2.log 2>&1; tail -1 gpurun_out/$tag/bench_cfg2.log
timeout 900 python bench.py --config cfg3 > gpurun_out/$tag/bench_cfg3.log 2>&1; tail -1 gpurun_out/$tag/bench_cfg3.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/$tag/bench_ref.log 2>&1; tail -1 gpurun_out/$tag/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$tag/ncu_bench_cfg4.log 2>&1
ls -la gpurun_out/$tag
