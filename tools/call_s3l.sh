D=gpurun_out/r2s3_l
mkdir -p $D
bash tools/call_ab.sh r2s3_l cfg4 > /dev/null 2>&1
timeout 600 python tools/tune_sweep.py --config cfg3 --runs 3 '{}' '{"joint_lanes_per_warp": 13}' '{"joint_lanes_per_warp": 14}' > $D/cfg3_sweep.log 2>&1
for k in 1 2; do timeout 900 python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 1 > $D/bench_cfg3_$k.log 2>&1; done
timeout 900 python bench.py --config cfg4 --no-cpu-baseline --e2e-steps 2 > $D/bench_cfg4.log 2>&1
