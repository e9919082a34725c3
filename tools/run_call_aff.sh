PADSIM_J_AFF=1 PADSIM_J_WPF=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/run_ab_env.sh cfg4 af4 "X=0" "PADSIM_J_AFF=1" "PADSIM_J_WPF=1" "PADSIM_J_AFF=1 PADSIM_J_WPF=1"
bash tools/run_ab_env.sh cfg3 af3 "X=0" "PADSIM_J_AFF=1" "PADSIM_J_WPF=1" "PADSIM_J_AFF=1 PADSIM_J_WPF=1"
