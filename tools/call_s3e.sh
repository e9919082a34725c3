D=gpurun_out/r2s3_e
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "launch_variants or static_records" > $D/tests.log 2>&1
bash tools/call_ab.sh r2s3_e cfg4 cfg2 > /dev/null 2>&1
AB_ARGS="" timeout 600 python tools/tune_sweep.py --config cfg4 --runs 2 '{"serialize": 1}' > $D/new_ser.log 2>&1
PADSIM_LIB=build/ab/libpadsim_base.so timeout 600 python tools/tune_sweep.py --config cfg4 --runs 2 '{"serialize": 1}' > $D/base_ser.log 2>&1
