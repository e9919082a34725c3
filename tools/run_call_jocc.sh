bash tools/run_ab_env.sh cfg4 jo4 "X=0" "PADSIM_J_OCC=6" "PADSIM_J_OCC=4" "PADSIM_J_OCC=3" "PADSIM_J_OCC=2"
