#!/usr/bin/env python3
"""Randomised distributed parity (torchrun, one rank per GPU): every iteration all ranks
draw the same random configuration (topology, budget, group size / scale format,
allocator, rounding, codebooks, size) and re-configure ONE communicator in place
(dq_ctx_set_config: the peer region regrows / re-shapes between ring and butterfly);
each output must equal the single-GPU simulated round bit for bit and agree across
ranks.  Prints one JSON line on rank 0; exit code 1 on any mismatch.

    torchrun --nproc-per-node N tools/dist_fuzz.py [--iters 120] [--seed 0]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=120)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rng = np.random.default_rng(args.seed)  # identical stream on every rank
    comm = dq.Communicator(dq.PipelineConfig(n_workers=world), rank, world)
    sim_ctx = dq.Context(dq.PipelineConfig(n_workers=world))
    fails, n_ok, n_inf = [], 0, 0
    for it in range(args.iters):
        topo = "butterfly" if (world & (world - 1)) == 0 and rng.random() < 0.4 else "ring"
        d = int(rng.integers(1, 1 << int(rng.integers(10, 21))))
        b = float(np.round(rng.uniform(2.2, 9.0), 3))
        fmt = rng.random()
        s, hier = (16, True) if fmt < 0.75 else (int(rng.choice([8, 32, 64])), bool(rng.random() < 0.5))
        alloc = str(rng.choice(["fast", "fast", "general", "fixed"]))
        cfg = dq.PipelineConfig(n_workers=world, budget_bits=b, group_size=s, hierarchical_scales=hier,
                                correlated=bool(rng.random() < 0.8), non_uniform=bool(rng.random() < 0.8),
                                variable_width=alloc != "fixed", fixed_width=int(rng.choice([2, 4, 8])),
                                allocator={"general": dq.KIND_GENERAL, "fast": dq.KIND_FAST,
                                           "fixed": dq.KIND_FIXED}[alloc],
                                topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING,
                                seed=dq.SharedSeed(int(rng.integers(0, 1 << 30)), int(rng.integers(0, 5))))
        gseed = int(rng.integers(0, 1 << 30))
        g = torch.Generator(device="cuda").manual_seed(gseed)
        T = (d + 255) // 256
        scale = torch.exp(float(rng.uniform(0, 5)) * torch.randn(T, device="cuda", generator=g))
        ws = [(torch.randn(T, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1)[:d].contiguous()
              for _ in range(world)]
        comm.ctx.set_config(cfg)
        case = {"it": it, "topo": topo, "d": d, "b": b, "s": s, "hier": hier, "alloc": alloc}
        try:
            out, _ = comm.allreduce(ws[rank])
            torch.cuda.synchronize()
            err = None
        except dq.InfeasibleBudget:
            err = "infeasible"
        errs = [None] * world
        dist.all_gather_object(errs, err)
        if any(e is not None for e in errs):
            if rank == 0:
                if all(e == "infeasible" for e in errs):
                    try:
                        sim_ctx.set_config(cfg)
                        dq.run_round(ws, cfg, ctx=sim_ctx, metrics=False)
                        fails.append({**case, "error": "device infeasible, simulation not"})
                    except dq.InfeasibleBudget:
                        n_inf += 1
                else:
                    fails.append({**case, "error": f"ranks disagree on errors: {errs}"})
            continue
        gathered = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        agree = all(torch.equal(gathered[0], t) for t in gathered)
        if rank == 0:
            sim_ctx.set_config(cfg)
            sim = dq.run_round(ws, cfg, ctx=sim_ctx, metrics=False)
            if agree and torch.equal(sim.synced, out):
                n_ok += 1
            else:
                fails.append({**case, "error": "mismatch", "ranks_agree": agree})
    if rank == 0:
        print(json.dumps({"world": world, "ok": not fails, "rounds": n_ok, "infeasible_agree": n_inf,
                          "fails": fails[:10]}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if not fails or rank != 0 else 1)


if __name__ == "__main__":
    main()
