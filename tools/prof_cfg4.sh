set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_v5_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench_cfg4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stageC -c 1 -o gpurun_out/r1_v5_stageC_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_stageC.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stageA -c 1 -o gpurun_out/r1_v5_stageA_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_stageA.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:joint -c 1 -o gpurun_out/r1_v5_joint_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_joint.log 2>&1
ls -la gpurun_out
