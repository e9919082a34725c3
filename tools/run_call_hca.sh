timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/run_ab_env.sh cfg4 hca4 "PADSIM_NO_HCA=1" "X=0"
bash tools/run_ab_env.sh cfg2 hca2 "PADSIM_NO_HCA=1" "X=0"
