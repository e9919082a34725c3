timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg3 e13 $L/libpadsim_base.so $L/libpadsim_e1.so
bash tools/run_ab.sh cfg4 e14 $L/libpadsim_base.so $L/libpadsim_e1.so
