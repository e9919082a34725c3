mkdir -p gpurun_out/b4
timeout 900 python bench.py > gpurun_out/b4/bench_cfg4.log 2>&1
tail -1 gpurun_out/b4/bench_cfg4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['cpu_baseline']['value'])"
