D=gpurun_out/r2s3_k
mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q -x > $D/gpu_tests_full.log 2>&1; tail -3 $D/gpu_tests_full.log > $D/gpu_tests.log
bash tools/call_ab.sh r2s3_k cfg3 cfg4 > /dev/null 2>&1
for c in cfg3 cfg2; do timeout 900 python bench.py --config $c > $D/bench_$c.log 2>&1; done
