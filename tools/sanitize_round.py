#!/usr/bin/env python3
"""Small rounds for compute-sanitizer (racecheck / synccheck / memcheck): ring and butterfly
simulated rounds (leaf with permutation slices, fused DAR, fused sink decode, DA, gather
decode, allocation kernels, asynchronous allocation incl. the host-finished path) and the
codec primitives, each checked bit-exact against the C oracle.  Exit 1 on a mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2602_08923_b200._lib import check, lib  # noqa: E402

port = Oracle("port")
ok = True
for n, topo, d, b, force in [(4, "ring", 1 << 14, 4.0, 0), (8, "butterfly", (1 << 13) + 77, 3.0, 0),
                             (3, "ring", 1 << 12, 5.0, 1)]:
    ws = [port.generate_worker(d, seed=9, sigma_log=4.0, rank=r) for r in range(n)]
    want = port.run_round(ws, port.round_cfg(n, b, topo, seed=1))
    cfg = dq.PipelineConfig(n_workers=n, budget_bits=b, seed=dq.SharedSeed(1, 0),
                            topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING)
    check(lib().dq_debug_force_host_alloc(force))
    got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg)
    check(lib().dq_debug_force_host_alloc(0))
    same = np.array_equal(got.synced.cpu().numpy().view(np.uint32), want["synced"].view(np.uint32))
    print(f"round n={n} {topo} d={d} b={b} force_host={force}: {'ok' if same else 'MISMATCH'}", flush=True)
    ok &= same
    # primitives: leaf + DAR of chunk 0 under slot 1 of 4
    w = np.array([8] * 3 + [4] * 5 + [2] * 9, np.uint8)
    v = ws[0][: w.size * 256]
    q = dq.QuantContext(dq.SharedSeed(1, 0), chunk_index=0, hop_slot=1, n_slots=4)
    c = dq.compress_chunk(torch.from_numpy(v).cuda(), w, dq.CodecConfig(), q, 0)
    r = dq.decompress_accumulate_recompress(c, torch.from_numpy(v).cuda(), dq.CodecConfig(), q, 0)
    cc = port.codec(16, 256, True, True)
    qc = port.qctx(1, 0, 0, 1, 4, True)
    a = port.compress_chunk(v, w, cc, qc) == dq.serialize_chunk(c)
    bb = port.dar_chunk(dq.serialize_chunk(c), v, cc, qc) == dq.serialize_chunk(r)
    print(f"primitives: compress {'ok' if a else 'MISMATCH'}, dar {'ok' if bb else 'MISMATCH'}", flush=True)
    ok &= a and bb
torch.cuda.synchronize()
print("ALL OK" if ok else "FAILED", flush=True)
sys.exit(0 if ok else 1)
