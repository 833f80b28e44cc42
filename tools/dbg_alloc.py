#!/usr/bin/env python3
"""Diagnose asynchronous allocations handed to the host (DQ_DEBUG_ALLOC=1 prints the reason)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_08923_b200 as dq
from bench import make_inputs
n, d = int(sys.argv[1]), int(sys.argv[2])
ws = [torch.from_numpy(w).cuda() for w in make_inputs(n, d, 4.0)]
cfg = dq.PipelineConfig(n_workers=n, budget_bits=4.0, seed=dq.SharedSeed(1, 0))
ctx = dq.Context(cfg)
for k in range(3):
    t0 = time.time()
    r = dq.run_round(ws, cfg, ctx=ctx, metrics=False)
    torch.cuda.synchronize()
    print(n, d, "round", k, f"{(time.time() - t0) * 1e3:.1f} ms", ctx.wait()["n8"], flush=True)
