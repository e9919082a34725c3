D=gpurun_out/r2s3_d
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dynamic_records_exact" > $D/tests.log 2>&1
timeout 900 python tools/tune_sweep.py --config cfg3 --runs 2 '{}' '{"joint_groups": 1}' '{"joint_groups": 2}' '{"joint_groups": 3}' '{"joint_groups": 4}' > $D/cfg3.log 2>&1
timeout 900 python tools/tune_sweep.py --config cfg4 --runs 2 '{}' '{"joint_groups": 2}' '{"joint_groups": 3}' '{"joint_groups": 4}' '{"serialize": 1}' '{"serialize": 1, "joint_groups": 2}' '{"serialize": 1, "joint_groups": 3}' '{"serialize": 1, "joint_groups": 4}' > $D/cfg4.log 2>&1
