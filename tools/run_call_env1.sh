bash tools/run_ab_env.sh cfg4 ev4 "X=0" "PADSIM_J_LPW=16" "PADSIM_J_LPW=24" "PADSIM_BL_MASK=20" "PADSIM_BL_MASK=22"
