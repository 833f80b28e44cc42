#!/usr/bin/env python3
"""Host enqueue time vs device time of small asynchronous rounds.

    python tools/host_overhead.py                      # simulated round, one GPU
    torchrun --nproc-per-node N tools/host_overhead.py # dq_allreduce, one rank per GPU

Per size: host_us = wall time of enqueuing K rounds (no sync) / K; dev_us = CUDA-event time
of the same K rounds / K.  host_us >= dev_us means the round is launch-bound on the host."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402
from bench import synth  # noqa: E402


def measure(fn, k=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    return (t1 - t0) / k * 1e6, a.elapsed_time(b) / k * 1e3


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        cfg = dq.PipelineConfig(n_workers=world, budget_bits=4.0, seed=dq.SharedSeed(1, 0))
        comm = dq.Communicator(cfg, rank, world)
    for e in (16, 18, 20, 22):
        d = 1 << e
        if world > 1:
            x = synth(torch, d, 1, 4.0, seed=rank + 1)[0]
            out = torch.empty_like(x)
            h, g = measure(lambda: comm.allreduce(x, out, async_op=True))
        else:
            cfg = dq.PipelineConfig(n_workers=4, budget_bits=4.0, seed=dq.SharedSeed(1, 0))
            ctx = dq.Context(cfg)
            xs = synth(torch, d, 4, 4.0)
            out = torch.empty(d, device="cuda")
            h, g = measure(lambda: dq.run_round(xs, cfg, out=out, ctx=ctx, metrics=False))
        if rank == 0:
            print(json.dumps({"world": world, "d": d, "host_us": round(h, 1), "dev_us": round(g, 1)}), flush=True)


if __name__ == "__main__":
    main()
