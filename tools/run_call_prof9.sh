tag=r1_v9
ncu --set full --clock-control none --import-source on -k regex:stageC -c 3 -o gpurun_out/${tag}_stageC_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_C.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stageA -c 1 -o gpurun_out/${tag}_stageA_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_A.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:joint -c 1 -o gpurun_out/${tag}_joint_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_J4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:joint -c 1 -o gpurun_out/${tag}_joint_cfg3 python tools/prof_run.py --config cfg3 --runs 1 > gpurun_out/ncu_${tag}_J3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_${tag}_bench.log 2>&1
ls -la gpurun_out/${tag}*
