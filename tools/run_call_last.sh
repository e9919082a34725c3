mkdir -p gpurun_out/last
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/last/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/last/bench_cfg4.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/last/bench_ref.log 2>&1
cat gpurun_out/last/gpu_tests.log; tail -1 gpurun_out/last/smoke.log; tail -1 gpurun_out/last/bench_cfg4.log | cut -c1-200; tail -1 gpurun_out/last/bench_ref.log | cut -c1-120
