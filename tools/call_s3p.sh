D=gpurun_out/r2s3_p
mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q -x > $D/gpu_tests_full.log 2>&1; tail -3 $D/gpu_tests_full.log > $D/gpu_tests.log
bash tools/call_ab.sh r2s3_p cfg4 cfg2 > /dev/null 2>&1
timeout 600 python tools/tune_sweep.py --config cfg4 --runs 2 '{"serialize": 1}' > $D/new_ser.log 2>&1
PADSIM_LIB=build/ab/libpadsim_base.so timeout 600 python tools/tune_sweep.py --config cfg4 --runs 2 '{"serialize": 1}' > $D/base_ser.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:'stageC' -o $D/mC python tools/prof_run.py --config cfg4 --runs 1 > $D/ncu_m.log 2>&1
python tools/ncu_summary.py full $D/mC.ncu-rep > $D/sum_mC.txt 2>&1
rm -f $D/*.ncu-rep
