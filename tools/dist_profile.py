#!/usr/bin/env python3
"""Per-kernel-family device time of distributed rounds (dq_profile: CUDA events around every
launch; the profiled rounds take the host-synchronous allocation path).

    torchrun --nproc-per-node N tools/dist_profile.py [--sizes 16,18,20]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402
from bench import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="16,18,20,24")
    ap.add_argument("--rounds", type=int, default=20)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = dq.PipelineConfig(n_workers=world, budget_bits=4.0, seed=dq.SharedSeed(1, 0))
    comm = dq.Communicator(cfg, rank, world)
    for e in (int(v) for v in args.sizes.split(",")):
        d = 1 << e
        x = synth(torch, d, 1, 4.0, seed=rank + 1)[0]
        out = torch.empty_like(x)
        for _ in range(3):
            comm.allreduce(x, out)
        comm.ctx.profile(True)
        comm.ctx.read_profile(reset=True)
        tot = 0.0
        for _ in range(args.rounds):
            _, info = comm.allreduce(x, out)
            tot += info["ms_total"]
        prof = comm.ctx.read_profile(reset=True)
        comm.ctx.profile(False)
        rec = {"rank": rank, "d": d, "round_us": round(tot / args.rounds * 1e3, 1),
               "families_us": {k: round(v["ms"] / args.rounds * 1e3, 1) for k, v in prof.items() if v["launches"]}}
        allr = [None] * world
        dist.all_gather_object(allr, rec)
        if rank == 0:
            for r in allr:
                print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
