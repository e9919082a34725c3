D=gpurun_out/r2s3_m
mkdir -p $D
for k in 1 2; do
  PADSIM_LIB=build/ab/libpadsim_base.so timeout 900 python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 1 > $D/bench_cfg3_base_$k.log 2>&1
  timeout 900 python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 1 > $D/bench_cfg3_new_$k.log 2>&1
done
timeout 600 python bench.py --config cfg1 --no-cpu-baseline --e2e-steps 1 > $D/bench_cfg1_new.log 2>&1
timeout 600 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py -q -x -k "wide or launch_variants" > $D/tests.log 2>&1
