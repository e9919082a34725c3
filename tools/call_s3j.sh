D=gpurun_out/r2s3_j
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "launch_variants or dynamic_records or cfg4_shape" > $D/tests.log 2>&1
bash tools/call_ab.sh r2s3_j cfg4 > /dev/null 2>&1
timeout 600 python tools/joint_balance.py --config cfg3 > $D/balance_cfg3.json 2>&1
timeout 900 python tools/tune_sweep.py --config cfg3 --runs 2 '{}' '{"joint_lanes_per_warp": 12}' '{"joint_lanes_per_warp": 10}' '{"joint_reg_cap": 1}' '{"joint_reg_cap": 1, "joint_lanes_per_warp": 8}' > $D/cfg3_sweep.log 2>&1
