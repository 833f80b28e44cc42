#!/usr/bin/env python3
"""DDP with the DynamiQ comm hook (torchrun, one rank per GPU): the hooked gradient
must be close to the exact mean gradient (vNMSE small) and identical on all ranks."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from torch.nn.parallel import DistributedDataParallel as DDP  # noqa: E402

from paper_2602_08923_b200.ddp import DynamiQHookState, dynamiq_hook  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(1024, 2048), torch.nn.GELU(), torch.nn.Linear(2048, 1024)).cuda()
    ref = torch.nn.Sequential(torch.nn.Linear(1024, 2048), torch.nn.GELU(), torch.nn.Linear(2048, 1024)).cuda()
    ref.load_state_dict(model.state_dict())
    ddp = DDP(model, device_ids=[local], bucket_cap_mb=4)
    ddp_ref = DDP(ref, device_ids=[local], bucket_cap_mb=4)
    ddp.register_comm_hook(DynamiQHookState(budget_bits=5.0), dynamiq_hook)
    torch.manual_seed(100 + rank)
    x = torch.randn(64, 1024, device="cuda")
    for m in (ddp, ddp_ref):
        m(x).pow(2).mean().backward()
    err = sum(float(((p.grad - q.grad) ** 2).sum()) for p, q in zip(model.parameters(), ref.parameters()))
    nrm = sum(float((q.grad ** 2).sum()) for q in ref.parameters())
    flat = torch.cat([p.grad.reshape(-1) for p in model.parameters()])
    allg = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(allg, flat)
    agree = all(torch.equal(allg[0], t) for t in allg)
    ok = agree and err / nrm < 1e-2
    if rank == 0:
        print(json.dumps({"world": world, "vnmse_vs_nccl_mean": err / nrm, "ranks_agree": agree, "ok": ok}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
