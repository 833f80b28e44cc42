#!/usr/bin/env python3
"""Minimal distributed small-round check (debugging aid): a few all-reduces at small d,
each synchronised and compared with the simulated round."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2602_08923_b200 as dq
from bench import synth

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
topo = os.environ.get("TOPO", "ring")
cfg = dq.PipelineConfig(n_workers=world, budget_bits=4.0, seed=dq.SharedSeed(1, 0),
                        topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING)
comm = dq.Communicator(cfg, rank, world)
for d in [int(v) for v in os.environ.get("SIZES", "65536").split(",")]:
    xs = synth(torch, d, world, 4.0, seed=3)
    for it in range(int(os.environ.get("ITERS", "2"))):
        t0 = time.time()
        out = comm.allreduce(xs[rank], async_op=True)
        torch.cuda.synchronize()
        sim = dq.run_round(xs, cfg, metrics=False).synced if rank == 0 else None
        ok = torch.equal(sim, out) if rank == 0 else None
        print(f"rank {rank} d {d} it {it} {time.time() - t0:.3f}s ok={ok}", flush=True)
dist.barrier()
dist.destroy_process_group()
