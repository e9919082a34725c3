D=gpurun_out/w7
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py -x -q -k "wide or large_nodes" > $D/wide_tests.log 2>&1; tail -3 $D/wide_tests.log
AB_ARGS="--traces 1 --cand-stride 8" bash tools/call_ab.sh w7 cfg5
