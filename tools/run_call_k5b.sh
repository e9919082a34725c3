timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/run_ab_env.sh cfg2 kb2 "PADSIM_KC5=1" "X=0"
bash tools/run_ab_env.sh cfg4 kb4 "PADSIM_KC3=1" "X=0"
