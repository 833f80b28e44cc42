#!/usr/bin/env python3
"""Message-size / budget / topology sweep (BASELINE configs 4 and 5), one rank per GPU.

    torchrun --nproc-per-node N tools/sweep.py [--sizes 18:30] [--budgets 2,3,4,6] [--topology ring,butterfly]

For every (topology, budget, d) it times the DynamiQ all-reduce (max over ranks,
CUDA events) and NCCL's bf16 all-reduce of the same d, and measures vNMSE of the
DynamiQ sum against the exact fp32 NCCL sum of the same inputs (heavy-tailed
locality gradients, sigma_log = 4).  Prints one JSON line per case on rank 0.
b = 2 is infeasible in the reference (payload budget 1.4375 < 2): reported as such.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402


def timed(fn, steps, st):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="18:30", help="lo:hi[:step] exponents of d")
    ap.add_argument("--budgets", default="4")
    ap.add_argument("--topology", default="ring")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--transport", default="peer", help="ring transport: peer | nccl")
    ap.add_argument("--sigma-log", type=float, default=4.0)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    parts = [int(x) for x in args.sizes.split(":")]
    lo, hi, step = parts[0], parts[1], parts[2] if len(parts) > 2 else 1
    st = torch.cuda.current_stream()
    for topo in args.topology.split(","):
        if topo == "butterfly" and world & (world - 1):
            continue
        for b in (float(x) for x in args.budgets.split(",")):
            cfg = dq.PipelineConfig(n_workers=world, budget_bits=b, seed=dq.SharedSeed(1, 0),
                                    topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING)
            comm = dq.Communicator(cfg, rank, world, transport=args.transport)
            for e in range(lo, hi + 1, step):
                d = 1 << e
                g = torch.Generator(device="cuda").manual_seed(1)
                T = (d + 255) // 256
                scale = torch.exp(args.sigma_log * torch.randn(T, device="cuda", generator=g))
                g.manual_seed(1000 + rank)
                x = (torch.randn(T, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1)[:d].contiguous()
                out = torch.empty_like(x)
                rec = {"topology": topo, "transport": comm.transport, "budget": b, "n_gpus": world, "d": d, "bytes_fp32": 4 * d}
                try:
                    ms = timed(lambda: comm.allreduce(x, out, async_op=True), args.steps, st)
                except dq.InfeasibleBudget as ex:
                    rec["infeasible"] = str(ex)
                    if rank == 0:
                        print(json.dumps(rec), flush=True)
                    break
                truth = x.clone()
                dist.all_reduce(truth)
                err = ((out.double() - truth.double()) ** 2).sum()
                ref = (truth.double() ** 2).sum()
                dist.all_reduce(err)
                xb = x.to(torch.bfloat16)
                nms = timed(lambda: dist.all_reduce(xb), args.steps, st)
                rec.update(ms=round(ms, 4), effective_gbs=round(4 * d / ms / 1e6, 2),
                           whole_job_gbs=round(world * 4 * d / ms / 1e6, 2), vnmse=float(err / world / ref),
                           nccl_bf16_ms=round(nms, 4), nccl_bf16_effective_gbs=round(4 * d / nms / 1e6, 2))
                if rank == 0:
                    print(json.dumps(rec), flush=True)
            del comm
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
