D=gpurun_out/r2s3_a
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $D/gpu_tests_full.log 2>&1; tail -5 $D/gpu_tests_full.log > $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
for c in cfg4 cfg3; do timeout 900 python bench.py --config $c > $D/bench_$c.log 2>&1; done
