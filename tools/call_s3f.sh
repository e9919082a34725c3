D=gpurun_out/r2s3_f
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_wide.py -q -x -k "forced" > $D/tests.log 2>&1
timeout 600 python tools/tune_sweep.py --config cfg1 --runs 5 '{}' '{"wide_path": 1}' > $D/cfg1.log 2>&1
timeout 600 python tools/tune_sweep.py --config cfg2 --runs 2 '{}' '{"wide_path": 1}' > $D/cfg2.log 2>&1
timeout 600 python tools/tune_sweep.py --config cfg3 --runs 2 '{}' '{"wide_path": 1}' > $D/cfg3.log 2>&1
