timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg4 k6 $L/libpadsim_base.so $L/libpadsim_k6.so
bash tools/run_ab.sh cfg2 k6b $L/libpadsim_base.so $L/libpadsim_k6.so
