L=paper_2601_12241_b200
bash tools/run_ab.sh cfg4 kp4 $L/libpadsim_p8.so $L/libpadsim_p16.so $L/libpadsim_p4.so
bash tools/run_ab.sh cfg2 kp2 $L/libpadsim_p8.so $L/libpadsim_p16.so $L/libpadsim_p4.so
