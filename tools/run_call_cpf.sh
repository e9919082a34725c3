timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg4 cpf4 $L/libpadsim_c0.so $L/libpadsim_c1.so
