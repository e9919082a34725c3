bash tools/run_ab_env.sh cfg3 lpw "PADSIM_J_LPW=16" "PADSIM_J_LPW=12" "PADSIM_J_LPW=10" "PADSIM_J_LPW=20" "PADSIM_J_LPW=24"
