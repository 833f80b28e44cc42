#!/usr/bin/env python3
"""Distributed parity check (run under torchrun, one rank per GPU).

Every rank builds the same n synthetic gradients (rank-keyed), all-reduces its
own with dq_allreduce (peer-memory ring and NCCL transports), and rank 0
compares the result bit for bit with the single-GPU simulated round over all n
gradients (itself pinned to the oracle by tests/test_gpu_round.py) and, at small
sizes, with the CPU oracle's run_round.  Prints one JSON line on rank 0;
exit code 1 on mismatch.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    results = {}
    ok = True
    only = os.environ.get("DIST_CHECK_TRANSPORTS", "peer,nccl").split(",")
    cases = [("ring", 1 << 16, 4.0, t) for t in only]
    cases += [("ring", (1 << 20) + 300, 5.0, t) for t in only]
    cases += [("butterfly", 1 << 16, 4.0, t) for t in only] + [("butterfly", (1 << 20) + 300, 3.0, t) for t in only]
    cases += [("butterfly", 1 << 24, 4.0, "peer"), ("butterfly", 3000, 6.0, "peer")]
    cases += [("ring", 1 << 24, 4.0, t) for t in only] + [("ring", 1 << 28, 4.0, t) for t in only]
    cases += [("ring", 3000, 6.0, "peer"), ("ring", 1 << 22, 2.6, "peer")]
    cases = [c + ({},) for c in cases]
    # ablation formats (generic kernels over NCCL) and the general allocator, on every rank
    flat32 = {"group_size": 32, "hierarchical_scales": False}
    cases += [("ring", 1 << 16, 5.0, "peer", flat32), ("butterfly", (1 << 18) + 77, 5.0, "peer", flat32),
              ("ring", 1 << 16, 4.0, "peer", {"allocator": dq.KIND_GENERAL}),
              ("ring", (1 << 20) + 5, 4.0, "peer", {"allocator": dq.KIND_GENERAL, "correlated": False})]
    if os.environ.get("DIST_CHECK_SMALL"):  # under compute-sanitizer: the small cases only
        cases = [c for c in cases if c[1] <= (1 << 16) + 300]
    comms = {}
    for topo, d, b, transport, extra in cases:
        if topo == "butterfly" and world & (world - 1):
            continue
        cfg = dq.PipelineConfig(n_workers=world, budget_bits=b, seed=dq.SharedSeed(3, 1),
                                topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING, **extra)
        g = torch.Generator(device="cuda").manual_seed(7)
        T = (d + 255) // 256
        scale = torch.exp(4.0 * torch.randn(T, device="cuda", generator=g))
        ws = [(torch.randn(T, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1)[:d].contiguous()
              for _ in range(world)]
        if rank == 0 and os.environ.get("DIST_CHECK_VERBOSE"):
            print(f"case {topo} {transport} d={d} b={b}", file=sys.stderr, flush=True)
        # peer-transport contexts are reused across sizes and budgets (region regrowth, epochs)
        key = (topo, transport, b, tuple(sorted(extra.items())))
        if key not in comms:
            comms[key] = dq.Communicator(cfg, rank, world, transport=transport)
        comm = comms[key]
        out, info = comm.allreduce(ws[rank])
        out2, _ = comm.allreduce(ws[rank])  # second round on the same context (buffer reuse)
        torch.cuda.synchronize()
        same_twice = bool(torch.equal(out, out2))
        # every rank must hold the identical sum
        gathered = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        ranks_agree = all(torch.equal(gathered[0], t) for t in gathered)
        if rank == 0:
            sim = dq.run_round(ws, cfg, ctx=dq.Context(cfg))
            match_sim = bool(torch.equal(sim.synced, out))
            rec = {"transport": comm.transport, "match_sim": match_sim, "ranks_agree": ranks_agree,
                   "same_twice": same_twice,
                   "u_equal": info["u"] == sim.u, "vnmse": sim.vnmse, "n8_4_2": [info["n8"], info["n4"], info["n2"]]}
            if d <= (1 << 16):
                from oracle.oracle import Oracle
                port = Oracle("port")
                okw = {"s": extra.get("group_size", 16), "hierarchical": extra.get("hierarchical_scales", True),
                       "correlated": extra.get("correlated", True),
                       "allocator": {0: "general", 1: "fast", 2: "fixed"}[extra.get("allocator", dq.KIND_FAST)]}
                want = port.run_round([w.cpu().numpy() for w in ws],
                                      port.round_cfg(world, b, topo, seed=3, rnd=1, **okw))
                rec["match_oracle"] = bool(np.array_equal(out.cpu().numpy().view(np.uint32),
                                                          want["synced"].view(np.uint32)))
            ok &= all(v for k, v in rec.items() if k.startswith("match") or k in ("ranks_agree", "same_twice"))
            ok &= rec["transport"] == transport
            tag = "".join(f"_{k}{v}" for k, v in sorted(extra.items()))
            results[f"{topo}_{transport}_d{d}_b{b}{tag}"] = rec
        dist.barrier()
    comms.clear()
    if rank == 0:
        print(json.dumps({"world": world, "ok": ok, "cases": results}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok or rank != 0 else 1)


if __name__ == "__main__":
    main()
