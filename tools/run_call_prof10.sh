tag=r1_v10
ncu --set full --clock-control none --import-source on -k regex:stageC --launch-skip 2 -c 1 -o gpurun_out/${tag}_stageC7_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_C7.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stageC --launch-skip 1 -c 1 -o gpurun_out/${tag}_stageC4_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_C4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stageC -c 1 -o gpurun_out/${tag}_stageC2_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_C2.log 2>&1
ls -la gpurun_out/${tag}*
