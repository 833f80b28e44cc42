#!/usr/bin/env python3
"""Randomised round parity: random configurations (workers, topology, budget, size,
scale format, allocator, rounding, codebooks, generator) run on the GPU and by the CPU
oracle; synced gradient, wire_hash, allocation and accounting must be identical.

    python tools/fuzz_rounds.py [--seconds 300] [--seed 0]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402
from oracle.oracle import Oracle, OracleError  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    port = Oracle("port")
    rng = np.random.default_rng(args.seed)
    t0 = time.time()
    n_ok = n_inf = n_async = 0
    fails = []
    while time.time() - t0 < args.seconds:
        topo = "butterfly" if rng.random() < 0.35 else "ring"
        n = int(2 ** rng.integers(1, 5)) if topo == "butterfly" else int(rng.integers(2, 13))
        d = int(rng.integers(1, 1 << int(rng.integers(8, 18))))
        b = float(np.round(rng.uniform(2.2, 9.0), 3))
        s = int(rng.choice([8, 16, 16, 16, 32, 64, 128]))
        hier = bool(rng.random() < 0.7)
        corr = bool(rng.random() < 0.8)
        nonu = bool(rng.random() < 0.8)
        alloc = str(rng.choice(["fast", "fast", "general", "fixed"]))
        fw = int(rng.choice([2, 4, 8]))
        kind = str(rng.choice(["locality", "iid"]))
        sig = float(rng.uniform(0, 6))
        seed = int(rng.integers(0, 1 << 31))
        # half the rounds without the wire hash: the asynchronous device allocation (§5a)
        wire = bool(rng.random() < 0.5)
        ws = [port.generate_worker(d, seed=seed, sigma_log=sig, rank=r, kind=kind) for r in range(n)]
        ocfg = port.round_cfg(n, b, topo, seed=seed & 0xffff, rnd=int(seed % 7), s=s, hierarchical=hier,
                              correlated=corr, non_uniform=nonu, variable_width=alloc != "fixed",
                              fixed_width=fw, allocator=alloc)
        case = dict(topo=topo, n=n, d=d, b=b, s=s, hier=hier, corr=corr, nonu=nonu, alloc=alloc, fw=fw,
                    kind=kind, sig=sig, seed=seed, wire=wire)
        try:
            want = port.run_round(ws, ocfg)
        except OracleError as e:
            want = e
        cfg = dq.PipelineConfig(n_workers=n, budget_bits=b, group_size=s, hierarchical_scales=hier,
                                correlated=corr, non_uniform=nonu, variable_width=alloc != "fixed",
                                fixed_width=fw,
                                allocator={"general": dq.KIND_GENERAL, "fast": dq.KIND_FAST,
                                           "fixed": dq.KIND_FIXED}[alloc],
                                topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING,
                                seed=dq.SharedSeed(seed & 0xffff, int(seed % 7)))
        try:
            got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg, collect_wire=wire,
                               with_allocation=True)
        except dq.DqError as e:
            if isinstance(want, OracleError) and want.code == e.code:
                n_inf += 1
                continue
            fails.append({**case, "error": f"device {type(e).__name__}: {e}; oracle {want}"})
            continue
        if isinstance(want, OracleError):
            fails.append({**case, "error": f"oracle raised {want}, device did not"})
            continue
        same = (np.array_equal(got.synced.cpu().numpy().view(np.uint32), want["synced"].view(np.uint32))
                and (not wire or got.wire_hash == want["wire_hash"]) and got.u == want["u"]
                and got.payload_bits == want["payload_bits"]
                and np.array_equal(got.widths, want["widths"]))
        if same:
            n_ok += 1
            n_async += not wire
        else:
            fails.append({**case, "error": "mismatch"})
    print(json.dumps({"ok": not fails, "rounds": n_ok, "async_rounds": n_async, "infeasible_agree": n_inf, "fails": fails[:10]}))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
