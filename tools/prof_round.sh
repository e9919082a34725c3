# usage: bash tools/prof_round.sh <tag>
tag=$1
ncu --set full --clock-control none --import-source on -k regex:stageC -c 1 -o gpurun_out/${tag}_stageC_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_C.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:joint -c 1 -o gpurun_out/${tag}_joint_cfg3 python tools/prof_run.py --config cfg3 --runs 1 > gpurun_out/ncu_${tag}_J.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stageA -c 1 -o gpurun_out/${tag}_stageA_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > gpurun_out/ncu_${tag}_A.log 2>&1
ls gpurun_out/${tag}*
