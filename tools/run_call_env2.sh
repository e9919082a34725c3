bash tools/run_ab_env.sh cfg4 e2_4 "X=0" "PADSIM_J_R168=0" "PADSIM_A_TB=128" "PADSIM_J_LPW=24"
