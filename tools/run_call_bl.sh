timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
PADSIM_BL_MASK=31 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
PADSIM_BL_MASK=31 PADSIM_KC5=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ctx_growth.py -m gpu -q -x 2>&1 | tail -2
bash tools/run_ab_env.sh cfg4 bl4 "PADSIM_BL_MASK=0" "PADSIM_BL_MASK=16" "PADSIM_BL_MASK=24" "PADSIM_BL_MASK=31"
bash tools/run_ab_env.sh cfg2 bl2 "PADSIM_BL_MASK=0" "PADSIM_BL_MASK=16" "PADSIM_BL_MASK=31"
