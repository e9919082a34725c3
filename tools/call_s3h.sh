D=gpurun_out/r2s3_h
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_config.py -q -x > $D/tests.log 2>&1
PADSIM_LIB=build/ab/libpadsim_base.so timeout 600 python tools/joint_balance.py --config cfg3 > $D/balance_cfg3.json 2>&1
PADSIM_LIB=build/ab/libpadsim_base.so timeout 600 python tools/joint_balance.py --config cfg4 > $D/balance_cfg4.json 2>&1
bash tools/call_ab.sh r2s3_h cfg3 cfg4 > /dev/null 2>&1
timeout 600 python tools/tune_sweep.py --config cfg3 --runs 2 '{}' '{"joint_lanes_per_warp": 8}' '{"joint_lanes_per_warp": 32}' > $D/cfg3_lpw_new.log 2>&1
