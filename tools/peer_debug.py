#!/usr/bin/env python3
"""One peer-transport round at a small size with a sync and a check after it (debug aid).

    torchrun --nproc-per-node 2 tools/peer_debug.py [d]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
    print(f"rank {rank}: can_access_peer", [torch.cuda.can_device_access_peer(local, q)
                                           for q in range(torch.cuda.device_count()) if q != local], flush=True)
    cfg = dq.PipelineConfig(n_workers=world, budget_bits=4.0, seed=dq.SharedSeed(3, 1))
    g = torch.Generator(device="cuda").manual_seed(7 + rank)
    x = torch.randn(d, device="cuda", generator=g)
    comm = dq.Communicator(cfg, rank, world, transport=os.environ.get("T", "peer"))
    for it in range(3):
        out, info = comm.allreduce(x)
        torch.cuda.synchronize()
        truth = x.clone()
        dist.all_reduce(truth)
        err = float(((out - truth) ** 2).sum() / (truth ** 2).sum())
        print(f"rank {rank} round {it}: transport={comm.transport} rel_err={err:.3e}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
