timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg3 pf3 $L/libpadsim_pf0.so $L/libpadsim_pf1.so
bash tools/run_ab.sh cfg4 pf4 $L/libpadsim_pf0.so $L/libpadsim_pf1.so
