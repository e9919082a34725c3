mkdir -p gpurun_out/b5
timeout 900 python bench.py > gpurun_out/b5/bench_cfg4.log 2>&1
timeout 900 python bench.py --config cfg2 > gpurun_out/b5/bench_cfg2.log 2>&1
timeout 900 python bench.py --config cfg3 > gpurun_out/b5/bench_cfg3.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b5/smoke.log 2>&1
for c in cfg4 cfg2 cfg3; do tail -1 gpurun_out/b5/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"; done; tail -1 gpurun_out/b5/smoke.log
