timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -m gpu -q -x 2>&1 | tail -2
L=paper_2601_12241_b200
bash tools/run_ab.sh cfg3 wx3 $L/libpadsim_base.so $L/libpadsim_wx.so
bash tools/run_ab.sh cfg3 wy3 $L/libpadsim_base.so $L/libpadsim_wx.so
bash tools/run_ab.sh cfg4 wx4 $L/libpadsim_base.so $L/libpadsim_wx.so
