PADSIM_A_TB=256 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/run_ab_env.sh cfg4 atb "PADSIM_A_TB=128" "PADSIM_A_TB=256"
