L=paper_2601_12241_b200
bash tools/run_ab.sh cfg4 kd4 $L/libpadsim_kd1.so $L/libpadsim_kd2.so
bash tools/run_ab.sh cfg2 kd2 $L/libpadsim_kd1.so $L/libpadsim_kd2.so
