D=gpurun_out/r2s3_c
mkdir -p $D
timeout 900 python tools/tune_sweep.py --config cfg4 --runs 3 '{}' '{"stage_c_batch_lists": 20}' '{"stage_c_batch_lists": 24}' '{"stage_c_batch_lists": 28}' '{"stage_c_batch_lists": 31}' '{"stage_c_batch_lists": 30}' > $D/bl_sweep.log 2>&1
timeout 600 python tools/tune_sweep.py --config cfg4 --runs 3 '{"serialize": 1}' '{"serialize": 1, "stage_c_batch_lists": 28}' '{"serialize": 1, "stage_c_batch_lists": 31}' > $D/bl_sweep_ser.log 2>&1
