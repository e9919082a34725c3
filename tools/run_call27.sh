python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/gpu_tests.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench22_cfg4.log 2>&1
python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench22_cfg2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stageC -c 1 -o gpurun_out/r1_v6_stageC_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_stageC6.log 2>&1
tail -4 gpurun_out/gpu_tests.log
