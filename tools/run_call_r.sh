L=paper_2601_12241_b200
bash tools/run_ab.sh cfg4 r4 $L/libpadsim_r168.so $L/libpadsim_r96.so $L/libpadsim_r80.so
bash tools/run_ab.sh cfg2 r2 $L/libpadsim_r168.so $L/libpadsim_r96.so $L/libpadsim_r80.so
