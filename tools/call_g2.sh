D=gpurun_out/g2
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jointg -c 1 -o $D/jg_cfg3 python tools/prof_run.py --config cfg3 --runs 1 > $D/ncu_J3.log 2>&1
{ python tools/ncu_summary.py full $D/jg_cfg3.ncu-rep; python tools/ncu_hot.py $D/jg_cfg3.ncu-rep 45; } > $D/sum_jg_cfg3.txt 2>&1
rm -f $D/*.ncu-rep
