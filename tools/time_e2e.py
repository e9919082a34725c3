import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench import build_workload
from workloads import DEFAULT_MODEL, get_config
import paper_2601_12241_b200 as pkg
from paper_2601_12241_b200.distributed import evaluate_sharded
cfg = get_config("cfg4")
role, cap, pols, traces, qps, cb = build_workload(cfg, 0, pkg.enumerate_pool_uniform)
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
stream = torch.cuda.current_stream(dev)
ctx = pkg.Context(0, stream.cuda_stream)
for k in range(4):
    t0 = time.perf_counter()
    out = evaluate_sharded(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"], ctx=ctx, device=0, cand_budget_w=cb)
    t1 = time.perf_counter()
    o2 = pkg.evaluate_allocations(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"], ctx=ctx, cand_budget_w=cb)
    t2 = time.perf_counter()
    print(f"evaluate_sharded {1e3*(t1-t0):.1f} ms   evaluate_allocations {1e3*(t2-t1):.1f} ms   device {ctx.replay_kernel_ms():.1f}")
