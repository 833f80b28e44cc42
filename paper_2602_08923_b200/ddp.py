"""PyTorch DDP communication hook running DynamiQ over the B200 C-ABI.

The paper deploys DynamiQ as a DDP comm hook (§4): every gradient
bucket is all-reduced with the compressed multi-hop protocol instead of NCCL's
all-reduce.  Usage:

    state = DynamiQHookState(budget_bits=4.0)       # one per process, after init_process_group
    ddp_model.register_comm_hook(state, dynamiq_hook)

Each call advances SharedSeed.round so successive rounds draw fresh shared
randomness (proj/include/dynamiq/random.hpp:12-15).  The hook returns the mean
(sum estimate / world size), like DDP's default all-reduce hook.
"""
import torch
import torch.distributed as dist

from .api import BUTTERFLY, RING, Communicator, PipelineConfig, SharedSeed


class DynamiQHookState:
    def __init__(self, budget_bits: float = 4.0, topology: str = "ring", seed: int = 1, group=None):
        self.world_size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.config = PipelineConfig(n_workers=self.world_size, budget_bits=budget_bits,
                                     topology=BUTTERFLY if topology == "butterfly" else RING,
                                     seed=SharedSeed(seed, 0))
        self.comm = Communicator(self.config, self.rank, self.world_size, group=group)
        self.round = 0
        self.last_info = {}

    def next_round(self) -> None:
        self.config.seed = SharedSeed(self.config.seed.seed, self.round)
        self.comm.ctx.set_config(self.config)
        self.round += 1


def dynamiq_hook(state: DynamiQHookState, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    buf = bucket.buffer()
    x = buf if buf.dtype == torch.float32 else buf.float()
    state.next_round()
    out, info = state.comm.allreduce(x.contiguous())
    state.last_info = info
    out.div_(state.world_size)
    if buf.dtype != torch.float32:
        out = out.to(buf.dtype)
    fut = torch.futures.Future()
    fut.set_result(out)
    return fut
