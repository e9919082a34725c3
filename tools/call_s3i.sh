D=gpurun_out/r2s3_i
mkdir -p $D
timeout 1800 python -m pytest tests -m gpu -q -x > $D/gpu_tests_full.log 2>&1; tail -3 $D/gpu_tests_full.log > $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
bash tools/call_ab.sh r2s3_i cfg4 cfg3 > /dev/null 2>&1
timeout 600 python tools/joint_balance.py --config cfg3 > $D/balance_cfg3.json 2>&1
for c in cfg4 cfg3; do timeout 900 python bench.py --config $c > $D/bench_$c.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:'stageC|joint|stageA' -o $D/m_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > $D/ncu_m.log 2>&1
python tools/ncu_traffic_update.py cfg4 r2s3_i_metrics $D/m_cfg4.ncu-rep > $D/traffic_update.log 2>&1
cp profiles/ncu_traffic.json $D/ncu_traffic.json
python tools/ncu_summary.py full $D/m_cfg4.ncu-rep > $D/sum_m_cfg4.txt 2>&1
rm -f $D/*.ncu-rep
