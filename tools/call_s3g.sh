D=gpurun_out/r2s3_g
mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q -x > $D/gpu_tests_full.log 2>&1; tail -5 $D/gpu_tests_full.log > $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
for c in cfg1 cfg3; do timeout 900 python bench.py --config $c > $D/bench_$c.log 2>&1; done
