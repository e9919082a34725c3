python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/gpu_tests.log
for v in default NO_PREFETCH BITS_GLOBAL; do
  if [ $v = default ]; then env=""; else env="PADSIM_$v=1"; fi
  env $env python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench17_cfg4_$v.log 2>&1
done
python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench17_cfg2.log 2>&1
tail -4 gpurun_out/gpu_tests.log
