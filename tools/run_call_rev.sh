bash tools/run_ab_env.sh cfg4 rev4 "X=0" "PADSIM_KC_REV=1"
bash tools/run_ab_env.sh cfg2 rev2 "X=0" "PADSIM_KC_REV=1"
