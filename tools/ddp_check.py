#!/usr/bin/env python3
"""DDP with the DynamiQ comm hook (torchrun, one rank per GPU).

Three training steps of a small MLP with the non-blocking hook (bucket all-reduces on the
hook's communication stream, no host synchronisation), then:
* bit-exact: every bucket's hooked gradient equals dq.run_round (the single-GPU simulated
  round, pinned to the oracle by tests/test_gpu_round.py) over the gathered per-rank
  buckets with the same SharedSeed round, divided by the world size;
* every rank holds identical gradients;
* the hooked gradient is close to the exact mean (vNMSE vs DDP's default NCCL hook).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from torch.nn.parallel import DistributedDataParallel as DDP  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402
from paper_2602_08923_b200.ddp import DynamiQHookState, dynamiq_hook  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.manual_seed(0)
    mk = lambda: torch.nn.Sequential(torch.nn.Linear(1024, 2048), torch.nn.GELU(),  # noqa: E731
                                     torch.nn.Linear(2048, 1024)).cuda()
    model, ref = mk(), mk()
    ref.load_state_dict(model.state_dict())
    ddp = DDP(model, device_ids=[local], bucket_cap_mb=4)
    ddp_ref = DDP(ref, device_ids=[local], bucket_cap_mb=4)
    state = DynamiQHookState(budget_bits=5.0, record=True)
    ddp.register_comm_hook(state, dynamiq_hook)
    vn = []
    for step in range(3):
        torch.manual_seed(100 + 10 * step + rank)
        x = torch.randn(64, 1024, device="cuda")
        for m in (ddp, ddp_ref):
            m.zero_grad(set_to_none=True)
            m(x).pow(2).mean().backward()
        err = sum(float(((p.grad - q.grad) ** 2).sum()) for p, q in zip(model.parameters(), ref.parameters()))
        nrm = sum(float((q.grad ** 2).sum()) for q in ref.parameters())
        vn.append(err / nrm)
    torch.cuda.synchronize()
    flat = torch.cat([p.grad.reshape(-1) for p in model.parameters()])
    allg = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(allg, flat)
    agree = all(torch.equal(allg[0], t) for t in allg)
    # bit-exact per bucket against the simulated round over the gathered inputs
    exact = []
    sim_ctx = None
    for rnd, xin, out in state.log:
        gathered = [torch.empty_like(xin) for _ in range(world)]
        dist.all_gather(gathered, xin)
        if rank == 0:
            cfg = dq.PipelineConfig(n_workers=world, budget_bits=5.0, seed=dq.SharedSeed(1, rnd))
            sim_ctx = sim_ctx or dq.Context(cfg)
            want = dq.run_round(gathered, cfg, ctx=sim_ctx, metrics=False).synced.div_(world)
            exact.append(bool(torch.equal(want, out)))
    ok = agree and max(vn) < 1e-2 and (rank != 0 or (exact and all(exact)))
    if rank == 0:
        print(json.dumps({"world": world, "buckets": len(state.log), "bit_exact_vs_sim_round": exact,
                          "vnmse_vs_nccl_mean": vn, "ranks_agree": agree, "ok": ok}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
