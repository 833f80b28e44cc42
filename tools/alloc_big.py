#!/usr/bin/env python3
"""Large-T allocation check (device vs oracle) + a d = 2^30 round smoke."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

port = Oracle("port")
rng = np.random.default_rng(0)
for T in (1 << 20, 1 << 21, 1 << 22, (1 << 22) + 12345):
    F = (np.exp(8 * rng.standard_normal(T)) * 256).astype(np.float32)
    w, p, u, pay = port.allocate_fast(F, 4.0)
    try:
        got = dq.allocate_fast(torch.from_numpy(F).cuda(), 4.0)
        ok = (np.array_equal(got.widths.cpu().numpy(), w) and
              np.array_equal(got.permutation.cpu().numpy().astype(np.uint32), p) and got.u == u)
        print("T", T, "ok", ok, got.u, u, got.counts, pay, got.payload_bits, flush=True)
    except Exception as e:
        print("T", T, "EXC", repr(e), "oracle u", u, pay, flush=True)
for d in (1 << 28, 1 << 29, 1 << 30):
    g = torch.Generator(device="cuda").manual_seed(1)
    T = d // 256
    scale = torch.exp(4.0 * torch.randn(T, device="cuda", generator=g))
    ws = [(torch.randn(T, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1) for _ in range(2)]
    try:
        r = dq.run_round(ws, dq.PipelineConfig(n_workers=2, budget_bits=4.0), metrics=False)
        torch.cuda.synchronize()
        print("d", d, "ok", r.info["n8"], r.info["n4"], r.info["n2"], r.u, flush=True)
    except Exception as e:
        print("d", d, "EXC", repr(e), flush=True)
    del ws
    torch.cuda.empty_cache()
