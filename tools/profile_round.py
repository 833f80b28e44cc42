#!/usr/bin/env python3
"""Run a few simulated rounds (for ncu / compute-sanitizer): python tools/profile_round.py [d] [n] [rounds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402
from bench import synth  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = dq.PipelineConfig(n_workers=n, budget_bits=4.0, seed=dq.SharedSeed(1, 0))
ws = synth(torch, d, n, 4.0)
for _ in range(rounds):
    r = dq.run_round(ws, cfg, metrics=False)
torch.cuda.synchronize()
print("ok", r.info["ms_total"], r.info["n8"], r.info["n4"], r.info["n2"])
