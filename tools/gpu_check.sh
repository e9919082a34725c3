#!/bin/bash
# One GPU evidence pass (run under gpurun): GPU tests, bench lines, 2-rank path.
#   bash tools/gpu_check.sh <tag> [configs...]
tag=$1; shift
cfgs=${@:-cfg4 cfg3}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu.txt
python -c "from paper_2601_12241_b200.build import build; build()" > $out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -25 > $out/gpu_tests.log
tail -3 $out/gpu_tests.log
for c in $cfgs; do
  timeout 900 python bench.py --config $c > $out/bench_$c.log 2>&1; tail -c 3000 $out/bench_$c.log | tail -1 | cut -c1-400
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --backend gloo --same-device --config cfg2 --steps 3 --e2e-steps 1 \
  > $out/bench_cfg2_2rank_gloo.log 2>&1; tail -1 $out/bench_cfg2_2rank_gloo.log | cut -c1-300
