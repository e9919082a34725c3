D=gpurun_out/w3
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_wide.py -x -q > $D/wide_tests.log 2>&1; tail -3 $D/wide_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stageC_wide -c 1 -o $D/cw_cfg5 python tools/prof_run.py --config cfg5 --traces 1 --cand-stride 16 --runs 1 > $D/ncu_cw.log 2>&1
{ python tools/ncu_summary.py full $D/cw_cfg5.ncu-rep; python tools/ncu_hot.py $D/cw_cfg5.ncu-rep 40; } > $D/sum_cw_cfg5.txt 2>&1
rm -f $D/*.ncu-rep
head -60 $D/sum_cw_cfg5.txt
