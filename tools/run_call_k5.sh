timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg4 k4 $L/libpadsim_k3.so $L/libpadsim.so
bash tools/run_ab.sh cfg2 k2 $L/libpadsim_k3.so $L/libpadsim.so
