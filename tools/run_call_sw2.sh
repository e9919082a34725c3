bash tools/run_ab_env.sh cfg3 sy3 "X=0" "PADSIM_SYNC_WIN=8" "PADSIM_SYNC_WIN=32"
bash tools/run_ab_env.sh cfg4 sy4 "X=0" "PADSIM_SYNC_WIN=8" "PADSIM_SYNC_WIN=32"
