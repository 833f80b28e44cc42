#!/usr/bin/env python3
"""Phase times of the one-CTA allocation (DQ_LIB_VARIANT=phases: -DDQ_SMALL_PHASES=1 prints
them from the kernel) at a few small sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_08923_b200 as dq
from bench import synth
for d in (1 << 16, 1 << 18, 1 << 19, 1 << 20):
    cfg = dq.PipelineConfig(n_workers=4, budget_bits=4.0, seed=dq.SharedSeed(1, 0))
    ws = synth(torch, d, 4, 4.0)
    ctx = dq.Context(cfg)
    for _ in range(3):
        dq.run_round(ws, cfg, ctx=ctx, metrics=False)
    torch.cuda.synchronize()
    ctx.close()
