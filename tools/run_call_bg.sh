PADSIM_BITS_GLOBAL_BIG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
bash tools/run_ab_env.sh cfg4 bg "X=0" "PADSIM_BITS_GLOBAL_BIG=1"
