D=gpurun_out/r2s3_b
mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or bench_config or boundary or ctx" > $D/gpu_tests.log 2>&1
PADSIM_LIB=build/ab/libpadsim_base.so timeout 300 python tools/stagec_balance.py --config cfg4 > $D/balance_base.log 2>&1
timeout 300 python tools/stagec_balance.py --config cfg4 > $D/balance_new.log 2>&1
bash tools/call_ab.sh r2s3_b cfg4 cfg2 > /dev/null 2>&1
