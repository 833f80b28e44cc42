#!/usr/bin/env python3
"""Diagnose host-finished allocations of small (one-CTA) asynchronous rounds."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2602_08923_b200 as dq
from oracle.oracle import Oracle
port = Oracle("port")
from paper_2602_08923_b200._lib import check, lib
cases = [(4, 1 << 21, 35, 0), (4, 1 << 21, 35, 2), (2, (1 << 20) + 256, 33, 0), (2, (1 << 20) + 256, 33, 2)]
for n, d, seed, force in cases:
    ws = [port.generate_worker(d, seed=seed, sigma_log=4.0, rank=r) for r in range(n)]
    cfg = dq.PipelineConfig(n_workers=n, budget_bits=4.0, seed=dq.SharedSeed(1, 0))
    ctx = dq.Context(cfg)
    check(lib().dq_debug_force_host_alloc(force))
    r = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg, ctx=ctx, with_allocation=True)
    check(lib().dq_debug_force_host_alloc(0))
    want = port.run_round(ws, port.round_cfg(n, 4.0, "ring", seed=1))
    ok = np.array_equal(r.synced.cpu().numpy().view(np.uint32), want["synced"].view(np.uint32))
    print(n, d, seed, force, "ok" if ok else "MISMATCH", ctx.host_allocations(), flush=True)
    ctx.close()
