timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg3 sl3 $L/libpadsim_base.so $L/libpadsim_sl.so
bash tools/run_ab.sh cfg4 sl4 $L/libpadsim_base.so $L/libpadsim_sl.so
bash tools/run_ab.sh cfg2 sl2 $L/libpadsim_base.so $L/libpadsim_sl.so
