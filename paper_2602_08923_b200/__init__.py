"""B200-native DynamiQ compressed multi-hop all-reduce (arXiv 2602.08923).

The compute path is the native library ``libdynamiq_b200.so`` (hand-written
sm_100a CUDA kernels + C++ runtime + NCCL over NVLink) behind the C-ABI in
``include/dynamiq_b200.h``.  This package is the Python mirror of the
reference's C++ interface for that path; see ``api.py``.
"""
from ._lib import (CudaError, DqError, InfeasibleBudget, InvalidArgument, MalformedBuffer,  # noqa: F401
                   NcclError, build, lib)
from .api import (BUTTERFLY, KIND_FAST, KIND_FIXED, KIND_GENERAL, RING, BitAllocation, CodecConfig,  # noqa: F401
                  Communicator, Context, DeviceChunk, FastAllocatorState, PipelineConfig, QuantContext,
                  RoundResult, SharedSeed, ablation_ladder, allocate_fast, allocate_fast_stateful, allocate_general, chunk_bytes, compress_chunk, compressed_size_bits, compute_stats,
                  decompress_accumulate, decompress_accumulate_recompress, decompress_chunk, parse_chunk,
                  reduce_stats, run_round, run_round_host, schedule, serialize_chunk, soa_from_reference, wire_bytes)

__version__ = "0.1.0"
