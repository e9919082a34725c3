D=gpurun_out/w1
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > $D/wide_tests.log 2>&1; tail -30 $D/wide_tests.log
timeout 600 python -m pytest tests -m gpu -x -q > $D/gpu_tests.log 2>&1; tail -3 $D/gpu_tests.log
