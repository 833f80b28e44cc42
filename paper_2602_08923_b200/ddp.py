"""PyTorch DDP communication hook running DynamiQ over the B200 C-ABI.

The paper deploys DynamiQ as a DDP comm hook (§4, 597-598): every gradient
bucket is all-reduced with the compressed multi-hop protocol instead of NCCL's
all-reduce.  Usage:

    state = DynamiQHookState(budget_bits=4.0)       # one per process, after init_process_group
    ddp_model.register_comm_hook(state, dynamiq_hook)

Non-blocking: the hook enqueues the bucket's all-reduce on a dedicated communication
stream (ordered after the bucket is ready on the caller's stream) and returns a
CUDA-aware Future whose completion is an event on that stream, so backward keeps
computing while the round runs and no host thread ever waits for the GPU.  The round
itself never synchronises with the host (the bit allocation is decided on the device,
dq_allreduce with info = NULL).

Each call advances SharedSeed.round so successive rounds draw fresh shared randomness
(proj/include/dynamiq/random.hpp:12-15).  The hook returns the mean (sum estimate /
world size), like DDP's default all-reduce hook.
"""
import torch
import torch.distributed as dist

from .api import BUTTERFLY, RING, Communicator, PipelineConfig, SharedSeed


class DynamiQHookState:
    def __init__(self, budget_bits: float = 4.0, topology: str = "ring", seed: int = 1, group=None,
                 record: bool = False):
        self.world_size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.config = PipelineConfig(n_workers=self.world_size, budget_bits=budget_bits,
                                     topology=BUTTERFLY if topology == "butterfly" else RING,
                                     seed=SharedSeed(seed, 0))
        self.comm = Communicator(self.config, self.rank, self.world_size, group=group)
        self.stream = torch.cuda.Stream()
        self.round = 0
        # record=True keeps (round, input, output) of every bucket for parity checks
        self.record = record
        self.log = []

    def next_round(self) -> int:
        r = self.round
        self.config.seed = SharedSeed(self.config.seed.seed, r)
        self.comm.ctx.set_config(self.config)
        self.round += 1
        return r


def dynamiq_hook(state: DynamiQHookState, bucket: dist.GradBucket) -> torch.futures.Future[torch.Tensor]:
    buf = bucket.buffer()
    caller = torch.cuda.current_stream()
    rnd = state.next_round()
    s = state.stream
    s.wait_stream(caller)  # the bucket's gradients are complete on the caller's stream
    fut = torch.futures.Future(devices=[buf.device])
    with torch.cuda.stream(s):
        x = buf if buf.dtype == torch.float32 else buf.float()
        x = x.contiguous()
        out = state.comm.allreduce(x, async_op=True)
        out.div_(state.world_size)
        if buf.dtype != torch.float32:
            out = out.to(buf.dtype)
        if state.record:
            state.log.append((rnd, x.clone(), out.clone()))
        buf.record_stream(s)
        out.record_stream(caller)
        fut.set_result(out)  # completion = an event on s; DDP's stream waits for it, the host does not
    return fut
