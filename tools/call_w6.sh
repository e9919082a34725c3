D=gpurun_out/w6
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_wide.py -x -q > $D/wide_tests.log 2>&1; tail -3 $D/wide_tests.log
AB_ARGS="--traces 1 --cand-stride 8" bash tools/call_ab.sh w6 cfg5
