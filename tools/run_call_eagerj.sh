timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg3 ej3 $L/libpadsim_j0.so $L/libpadsim_j1.so
bash tools/run_ab.sh cfg4 ej4 $L/libpadsim_j0.so $L/libpadsim_j1.so
