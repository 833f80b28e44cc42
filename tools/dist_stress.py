#!/usr/bin/env python3
"""Back-to-back asynchronous all-reduces on one communicator (torchrun, one rank per GPU).

Enqueues R rounds without any host synchronisation between them — alternating sizes,
so the peer region regrows, epochs advance and round parities alternate while earlier
rounds may still be running — keeping every output in its own buffer; then checks
each output bit for bit against the single-GPU simulated round of the same inputs and
across ranks.  Prints one JSON line on rank 0; exit code 1 on any mismatch.
"""
import json
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
    ok = True
    res = {}
    for topo in ("ring", "butterfly"):
        if topo == "butterfly" and world & (world - 1):
            continue
        cfg = dq.PipelineConfig(n_workers=world, budget_bits=4.0, seed=dq.SharedSeed(11, 2),
                                topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING)
        comm = dq.Communicator(cfg, rank, world)
        sizes = [(1 << 16) + 7, 1 << 20, 3000, (1 << 22) + 300, 1 << 18, 1 << 22, (1 << 16) + 7, 1 << 21] * 3
        inputs, outs = [], []
        for k, d in enumerate(sizes):
            g = torch.Generator(device="cuda").manual_seed(1000 * k + 17)
            T = (d + 255) // 256
            scale = torch.exp(3.0 * torch.randn(T, device="cuda", generator=g))
            ws = [(torch.randn(T, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1)[:d].contiguous()
                  for _ in range(world)]
            inputs.append(ws)
        torch.cuda.synchronize()
        dist.barrier()
        for k, d in enumerate(sizes):  # no host sync in between
            out = comm.allreduce(inputs[k][rank], async_op=True)
            outs.append(out)
        torch.cuda.synchronize()
        bad = []
        for k, d in enumerate(sizes):
            gathered = [torch.empty_like(outs[k]) for _ in range(world)]
            dist.all_gather(gathered, outs[k])
            agree = all(torch.equal(gathered[0], t) for t in gathered)
            match = True
            if rank == 0:
                sim = dq.run_round(inputs[k], cfg, ctx=dq.Context(cfg), metrics=False)
                match = bool(torch.equal(sim.synced, outs[k]))
            if not (agree and match):
                bad.append(k)
        res[topo] = {"rounds": len(sizes), "transport": comm.transport, "bad": bad}
        ok &= not bad
        del comm
        dist.barrier()
    if rank == 0:
        print(json.dumps({"world": world, "ok": ok, "cases": res}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok or rank != 0 else 1)


if __name__ == "__main__":
    main()
