D=gpurun_out/w5
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:joint -c 1 -o $D/j64_cfg5 python tools/prof_run.py --config cfg5 --traces 1 --cand-stride 64 --runs 1 --tuning '{"wide_path": 0}' > $D/ncu_j64.log 2>&1
{ python tools/ncu_summary.py full $D/j64_cfg5.ncu-rep; python tools/ncu_hot.py $D/j64_cfg5.ncu-rep 30; } > $D/sum_j64_cfg5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stageC_wide -c 1 -o $D/cw_cfg5 python tools/prof_run.py --config cfg5 --traces 1 --cand-stride 64 --runs 1 > $D/ncu_cw.log 2>&1
{ python tools/ncu_summary.py full $D/cw_cfg5.ncu-rep; python tools/ncu_hot.py $D/cw_cfg5.ncu-rep 40; } > $D/sum_cw_cfg5.txt 2>&1
rm -f $D/*.ncu-rep
head -30 $D/sum_j64_cfg5.txt; head -30 $D/sum_cw_cfg5.txt
