mkdir -p gpurun_out/b6
timeout 900 python bench.py --config cfg3 > gpurun_out/b6/bench_cfg3.log 2>&1
tail -1 gpurun_out/b6/bench_cfg3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
