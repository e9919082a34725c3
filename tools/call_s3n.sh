D=gpurun_out/r2s3_n
mkdir -p $D
timeout 600 python tools/tune_sweep.py --config cfg3 --runs 3 '{}' '{"joint_lanes_per_warp": 16}' > $D/sweep.log 2>&1
timeout 600 python tools/tune_sweep.py --flush --config cfg3 --runs 3 '{}' '{"joint_lanes_per_warp": 16}' > $D/sweep_flush.log 2>&1
timeout 900 python bench.py --config cfg3 --no-cpu-baseline --e2e-steps 1 > $D/bench_cfg3.log 2>&1
