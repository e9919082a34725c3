timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/run_ab_env.sh cfg4 w4 "X=0"
bash tools/run_ab_env.sh cfg3 w3 "X=0"
bash tools/run_ab_env.sh cfg2 w2 "X=0"
