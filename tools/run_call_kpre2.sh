timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg4 kq4 $L/libpadsim_p4.so $L/libpadsim_p2.so
bash tools/run_ab.sh cfg2 kq2 $L/libpadsim_p4.so $L/libpadsim_p2.so
