# Round-end evidence on one box: bash tools/run_final.sh <tag>
tag=$1
D=gpurun_out/$tag
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $D/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $D/gpu_tests_full.log 2>&1; tail -5 $D/gpu_tests_full.log > $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
for c in cfg4 cfg2 cfg3 cfg1; do
  timeout 900 python bench.py --config $c > $D/bench_$c.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $D/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $D/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stageC -c 5 -o $D/stageC_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > $D/ncu_C.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stageA -c 1 -o $D/stageA_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > $D/ncu_A.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:joint -c 1 -o $D/joint_cfg4 python tools/prof_run.py --config cfg4 --runs 1 > $D/ncu_J4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:joint -c 1 -o $D/joint_cfg3 python tools/prof_run.py --config cfg3 --runs 1 > $D/ncu_J3.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --backend gloo --same-device --config cfg2 --steps 2 --warmup 3 --no-cpu-baseline > $D/bench_cfg2_2rank_gloo.log 2>&1
timeout 2400 python bench.py --config cfg5 --steps 1 --warmup 3 --e2e-steps 1 --cpu-seconds 20 > $D/bench_cfg5.log 2>&1
# cfg5: the short metric list over every wide launch of one step (a --set full replay of a
# 30 s launch would take ~40 passes)
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:wide -o $D/wide_cfg5 python tools/prof_run.py --config cfg5 --runs 1 > $D/ncu_W5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stageC_wide -c 1 -o $D/cw_cfg5_sub python tools/prof_run.py --config cfg5 --traces 1 --cand-stride 16 --runs 1 > $D/ncu_cw.log 2>&1
# compute-sanitizer runs (tools/sanitize_small.py) are no longer allowed on this pool;
# the round-2 logs are in profiles/r2_sanitize/ and profiles/r2_final/san_summary.txt
# summaries on the box (the .ncu-rep files would exceed gpurun's 64 MiB copy-back)
{ python tools/ncu_summary.py full $D/stageC_cfg4.ncu-rep; python tools/ncu_hot.py $D/stageC_cfg4.ncu-rep 25; } > $D/sum_stageC_cfg4.txt 2>&1
{ python tools/ncu_summary.py full $D/stageA_cfg4.ncu-rep; python tools/ncu_hot.py $D/stageA_cfg4.ncu-rep 20; } > $D/sum_stageA_cfg4.txt 2>&1
{ python tools/ncu_summary.py full $D/joint_cfg4.ncu-rep; python tools/ncu_hot.py $D/joint_cfg4.ncu-rep 20; } > $D/sum_joint_cfg4.txt 2>&1
{ python tools/ncu_summary.py full $D/joint_cfg3.ncu-rep; python tools/ncu_hot.py $D/joint_cfg3.ncu-rep 20; } > $D/sum_joint_cfg3.txt 2>&1
{ python tools/ncu_summary.py full $D/cw_cfg5_sub.ncu-rep; python tools/ncu_hot.py $D/cw_cfg5_sub.ncu-rep 30; } > $D/sum_cw_cfg5_sub.txt 2>&1
echo '{}' > profiles/ncu_traffic.json
python tools/ncu_traffic_update.py cfg4 $tag $D/stageC_cfg4.ncu-rep $D/stageA_cfg4.ncu-rep $D/joint_cfg4.ncu-rep > /dev/null 2>&1
python tools/ncu_traffic_update.py cfg3 $tag $D/joint_cfg3.ncu-rep > /dev/null 2>&1
python tools/ncu_traffic_update.py cfg5 $tag $D/wide_cfg5.ncu-rep > /dev/null 2>&1
cp profiles/ncu_traffic.json $D/ncu_traffic.json
mkdir -p /tmp/ncu_keep && mv $D/*.ncu-rep /tmp/ncu_keep/ 2>/dev/null
ls -la $D
