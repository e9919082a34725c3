bash tools/run_ab_env.sh cfg4 wa4 "X=0" "PADSIM_JOINT_WITH_A=1" "PADSIM_JOINT_WITH_A=1 PADSIM_A_TB=128"
