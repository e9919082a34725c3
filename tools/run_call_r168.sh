PADSIM_J_R168=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/run_ab_env.sh cfg4 r168_4 "X=0" "PADSIM_J_R168=1"
bash tools/run_ab_env.sh cfg3 r168_3 "X=0" "PADSIM_J_R168=1"
