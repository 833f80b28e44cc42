#!/usr/bin/env python3
"""A distributed all-reduce captured in a CUDA graph (torchrun, one rank per GPU).

Every rank captures one dq_allreduce (peer transport: statistics exchange, device-side
allocation, fused hops over NVLink, gather decode; the round's epoch advances on the device)
and replays it on new inputs; each replay must equal the single-GPU simulated round over
the gathered inputs and agree across ranks.  Also times graph replays against direct
asynchronous calls (max over ranks, CUDA events).  One JSON line on rank 0."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402


def timed(fn, steps):
    st = torch.cuda.current_stream()
    for _ in range(3):
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
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok, res = True, {}
    sizes = [int(s) for s in os.environ.get("DIST_GRAPH_SIZES", f"{1 << 18},{(1 << 20) + 77}").split(",")]
    for topo in ("ring", "butterfly"):
        if topo == "butterfly" and world & (world - 1):
            continue
        cfg = dq.PipelineConfig(n_workers=world, budget_bits=4.0, seed=dq.SharedSeed(5, 0),
                                topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING)
        comm = dq.Communicator(cfg, rank, world)
        for d in sizes:
            x = torch.empty(d, device="cuda")
            out = torch.empty(d, device="cuda")
            g = torch.Generator(device="cuda").manual_seed(1 + rank)
            x.copy_(torch.randn(d, device="cuda", generator=g))
            comm.allreduce(x, out, async_op=True)  # sizes every buffer and region
            torch.cuda.synchronize()
            dist.barrier()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                comm.allreduce(x, out, async_op=True)
            bad = []
            for trial in range(3):
                g.manual_seed(100 * trial + rank)
                T = (d + 255) // 256
                scale = torch.exp(4.0 * torch.randn(T, device="cuda", generator=torch.Generator(device="cuda").manual_seed(trial)))
                x.copy_((torch.randn(T, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1)[:d])
                graph.replay()
                torch.cuda.synchronize()
                xs = [torch.empty_like(x) for _ in range(world)]
                dist.all_gather(xs, x)
                outs = [torch.empty_like(out) for _ in range(world)]
                dist.all_gather(outs, out)
                agree = all(torch.equal(outs[0], o) for o in outs)
                match = True
                if rank == 0:
                    sim = dq.run_round(xs, cfg, ctx=dq.Context(cfg), metrics=False)
                    match = bool(torch.equal(sim.synced, out))
                if not (agree and match):
                    bad.append(trial)
            direct_ms = timed(lambda: comm.allreduce(x, out, async_op=True), 50)
            graph_ms = timed(graph.replay, 50)
            xb = x.to(torch.bfloat16)
            nccl_ms = timed(lambda: dist.all_reduce(xb), 50)
            res[f"{topo}_d{d}"] = {"bad_replays": bad, "direct_ms": round(direct_ms, 4), "graph_ms": round(graph_ms, 4),
                                   "nccl_bf16_ms": round(nccl_ms, 4)}
            ok &= not bad
            del graph
        del comm
        dist.barrier()
    if rank == 0:
        print(json.dumps({"world": world, "ok": ok, "cases": res}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok or rank != 0 else 1)


if __name__ == "__main__":
    main()
