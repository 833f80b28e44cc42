"""Python mirror of the reference's hot-path interface, backed by the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference library
(``proj/include/dynamiq/{codec,stats,allocation,engine}.hpp``) so a caller of
``dynamiq::compress_chunk`` / ``run_round`` finds the same operations here:

=================================================  =============================================
reference (proj/include/dynamiq/...)               here
=================================================  =============================================
codec.hpp:64  compress_chunk                       :func:`compress_chunk`
codec.hpp:71  decompress_chunk                     :func:`decompress_chunk`
codec.hpp:75  decompress_accumulate                :func:`decompress_accumulate`
codec.hpp:86  decompress_accumulate_recompress     :func:`decompress_accumulate_recompress`
codec.hpp:94  serialize_chunk / parse_chunk        :func:`serialize_chunk` / :func:`parse_chunk`
codec.hpp:88  compressed_size_bits                 :func:`compressed_size_bits`
stats.hpp:19  compute_stats / reduce_stats         :func:`compute_stats` / :func:`reduce_stats`
allocation.hpp:63 allocate_fast (+permutation)     :func:`allocate_fast`
engine.hpp:63 run_round                            :func:`run_round` (all workers on one GPU)
(distributed run_round, PAPER §4)                  :class:`Communicator` ``.allreduce``
=================================================  =============================================

Tensors are torch CUDA tensors (device memory + the current stream are the
plumbing); all compute runs in the native library's sm_100a kernels.
Errors: :class:`InvalidArgument` (std::invalid_argument), :class:`InfeasibleBudget`,
:class:`MalformedBuffer` (std::runtime_error "malformed compressed buffer").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import (Config, InfeasibleBudget, InvalidArgument, MalformedBuffer, QCtx, RoundInfo,  # noqa: F401
                   check, lib)

RING, BUTTERFLY = 0, 1
KIND_GENERAL, KIND_FAST, KIND_FIXED = 0, 1, 2


@dataclass
class SharedSeed:
    """proj/include/dynamiq/random.hpp:12-15"""
    seed: int = 0
    round: int = 0


@dataclass
class QuantContext:
    """proj/include/dynamiq/codec.hpp:33-40"""
    seed: SharedSeed = field(default_factory=SharedSeed)
    chunk_index: int = 0
    hop_slot: int = 0
    n_slots: int = 1
    correlated: bool = True

    def _c(self) -> QCtx:
        return QCtx(self.seed.seed, self.seed.round, self.chunk_index, self.hop_slot, self.n_slots,
                    int(self.correlated))


@dataclass
class CodecConfig:
    """proj/include/dynamiq/codec.hpp:26-31 (device: S = 256, s in {8,16,32,64,128},
    hierarchical u8 + bf16 or flat bf16 group scales)"""
    group_size: int = 16
    super_group_size: int = 256
    hierarchical_scales: bool = True
    non_uniform: bool = True  # CodebookSet::non_uniform_defaults() vs uniform_all()

    def validate(self) -> None:
        if self.group_size == 0 or self.super_group_size % self.group_size or self.super_group_size % 4:
            raise InvalidArgument(2, "super-group size must be a positive multiple of the group size")
        if self.super_group_size != 256 or self.group_size not in (8, 16, 32, 64, 128):
            raise InvalidArgument(2, "device codec supports S=256 with s in {8, 16, 32, 64, 128}")


class _Format:
    """Scale format of this thread's chunk primitives for the duration of a call
    (dq_codec_format_set)."""

    def __init__(self, group_size: int = 16, hierarchical: bool = True):
        self.gs, self.hier = group_size, hierarchical

    def __enter__(self):
        pg, ph = C.c_uint32(), C.c_int()
        check(lib().dq_codec_format_set(self.gs, int(self.hier), C.byref(pg), C.byref(ph)))
        self.prev = (pg.value, ph.value)
        return self

    def __exit__(self, *exc):
        lib().dq_codec_format_set(self.prev[0], self.prev[1], None, None)


@dataclass
class PipelineConfig:
    """proj/include/dynamiq/engine.hpp:22-43 — same fields and defaults."""
    n_workers: int = 4
    group_size: int = 16
    super_group_size: int = 256
    budget_bits: float = 5.0
    non_uniform: bool = True
    variable_width: bool = True
    hierarchical_scales: bool = True
    correlated: bool = True
    fixed_width: int = 4
    allocator: int = KIND_FAST
    topology: int = RING
    codec: int = 0
    seed: SharedSeed = field(default_factory=lambda: SharedSeed(1, 0))
    threads: int = 1

    def _c(self) -> Config:
        return Config(self.n_workers, self.group_size, self.super_group_size, float(self.budget_bits),
                      int(self.non_uniform), int(self.variable_width), int(self.hierarchical_scales),
                      int(self.correlated), int(self.fixed_width), int(self.allocator), int(self.topology),
                      int(self.codec), self.seed.seed, self.seed.round, self.threads)


@dataclass
class DeviceChunk:
    """A compressed chunk resident in HBM (dq tiled SoA layout, include/dynamiq_b200.h).

    ``widths`` is implied by the run lengths (8, 4, 2, 16 order) like the
    reference's wire header (proj/src/codec.cpp:283-317); width 16 is the bf16
    passthrough record (codec.cpp:82-86)."""
    chunk_index: int
    n8: int
    n4: int
    n2: int
    data: torch.Tensor  # uint8, dq_chunk_bytes(n8, n4, n2, n16)
    n16: int = 0
    group_size: int = 16         # scale format (CodecConfig) the chunk was written with
    hierarchical: bool = True

    def fmt(self) -> _Format:
        return _Format(self.group_size, self.hierarchical)

    @property
    def n_sg(self) -> int:
        return self.n8 + self.n4 + self.n2 + self.n16

    @property
    def runs(self) -> tuple:
        return self.n8, self.n4, self.n2, self.n16

    @property
    def widths(self) -> np.ndarray:
        return np.array([8] * self.n8 + [4] * self.n4 + [2] * self.n2 + [16] * self.n16, np.uint8)


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None else 0)


def _runs(widths) -> tuple:
    """Run lengths of a width-sorted body; unsorted bodies are rejected like serialize_chunk
    (proj/src/codec.cpp:298-315)."""
    w = np.asarray(widths).astype(np.int64, copy=False).ravel()
    lut = np.full(256, -1, np.int64)
    lut[[8, 4, 2, 16]] = [0, 1, 2, 3]
    ok = (w >= 0) & (w < 256)
    cls = np.where(ok, lut[np.clip(w, 0, 255)], -1)
    bad = np.flatnonzero(cls < 0)
    if bad.size:
        raise InvalidArgument(2, f"unsupported codec width {int(w[bad[0]])}")
    if np.any(np.diff(cls) < 0):
        raise InvalidArgument(2, "chunk body must be ordered by width class 8,4,2,16")
    cnt = np.bincount(cls, minlength=4)
    return int(cnt[0]), int(cnt[1]), int(cnt[2]), int(cnt[3])


def _f32(t: torch.Tensor, n: int, what: str) -> torch.Tensor:
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise InvalidArgument(2, f"{what} must be a CUDA float32 tensor")
    if t.numel() != n:
        raise InvalidArgument(2, f"{what} length does not match chunk")
    t = t.contiguous()
    if t.data_ptr() % 16:
        t = t.clone()
    return t


def chunk_bytes(n8: int, n4: int, n2: int, n16: int = 0, cfg: Optional[CodecConfig] = None) -> int:
    """Device chunk bytes (dq tiled SoA) in cfg's scale format (default s=16 hierarchical)."""
    with _fmt_of(cfg):
        return lib().dq_chunk_bytes(n8, n4, n2, n16)


def wire_bytes(n8: int, n4: int, n2: int, n16: int = 0, cfg: Optional[CodecConfig] = None) -> int:
    """Reference serialize_chunk bytes incl. the 24-byte header (codec.cpp:268-291)."""
    with _fmt_of(cfg):
        return lib().dq_wire_bytes(n8, n4, n2, n16)


def _fmt_of(cfg: Optional[CodecConfig]) -> _Format:
    return _Format() if cfg is None else _Format(cfg.group_size, cfg.hierarchical_scales)


def compressed_size_bits(widths, S: int = 256, s: int = 16, hierarchical_scales: bool = True) -> int:
    """Exact reference wire size, header included (proj/src/codec.cpp:281-291)."""
    w = np.asarray(widths, np.uint8)
    scales = (16 + (S // s) * 8) if hierarchical_scales else (S // s) * 16
    return 192 + int(sum(int(x) * S + (0 if x == 16 else scales) for x in w.tolist()))


def compress_chunk(values: torch.Tensor, widths, cfg: CodecConfig, qctx: QuantContext,
                   first_sg_index: int = 0) -> DeviceChunk:
    cfg.validate()
    n8, n4, n2, n16 = _runs(widths)
    v = _f32(values, (n8 + n4 + n2 + n16) * 256, "chunk")
    out = torch.empty(max(chunk_bytes(n8, n4, n2, n16, cfg), 1), dtype=torch.uint8, device=v.device)
    q = qctx._c()
    with _fmt_of(cfg):
        check(lib().dq_compress_chunk(_ptr(v), n8, n4, n2, n16, C.byref(q), first_sg_index, int(cfg.non_uniform),
                                      _ptr(out), _stream()))
    return DeviceChunk(qctx.chunk_index, n8, n4, n2, out, n16, cfg.group_size, cfg.hierarchical_scales)


def decompress_accumulate_recompress(chunk: DeviceChunk, local: torch.Tensor, cfg: CodecConfig,
                                     qctx: QuantContext, first_sg_index: int = 0) -> DeviceChunk:
    cfg.validate()
    loc = _f32(local, chunk.n_sg * 256, "local buffer")
    out = torch.empty_like(chunk.data)
    q = qctx._c()
    with _fmt_of(cfg):
        check(lib().dq_dar_chunk(_ptr(chunk.data), _ptr(loc), *chunk.runs, C.byref(q),
                                 first_sg_index, int(cfg.non_uniform), _ptr(out), _stream()))
    return DeviceChunk(qctx.chunk_index, chunk.n8, chunk.n4, chunk.n2, out, chunk.n16, cfg.group_size,
                       cfg.hierarchical_scales)


def decompress_accumulate(chunk: DeviceChunk, acc: torch.Tensor, cfg: CodecConfig) -> None:
    """acc += decompress(chunk), in place (acc must be contiguous and 16-byte aligned)."""
    cfg.validate()
    if not (acc.is_cuda and acc.dtype == torch.float32 and acc.is_contiguous() and acc.data_ptr() % 16 == 0):
        raise InvalidArgument(2, "accumulator must be a contiguous, aligned CUDA float32 tensor")
    if acc.numel() != chunk.n_sg * 256:
        raise InvalidArgument(2, "accumulator length does not match chunk")
    with _fmt_of(cfg):
        check(lib().dq_da_chunk(_ptr(chunk.data), _ptr(acc), *chunk.runs, int(cfg.non_uniform),
                                _stream()))


def decompress_chunk(chunk: DeviceChunk, cfg: CodecConfig, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    cfg.validate()
    if out is None:
        out = torch.empty(chunk.n_sg * 256, dtype=torch.float32, device=chunk.data.device)
    elif out.numel() != chunk.n_sg * 256:
        raise InvalidArgument(2, "output length does not match chunk")
    with _fmt_of(cfg):
        check(lib().dq_decompress_chunk(_ptr(chunk.data), _ptr(out), *chunk.runs,
                                        int(cfg.non_uniform), _stream()))
    return out


def serialize_chunk(chunk: DeviceChunk, device: bool = False):
    """Reference wire bytes (proj/src/codec.cpp:319-343): host ``bytes``, or with
    ``device=True`` a CUDA uint8 tensor serialized on the GPU (dq_serialize_chunk)."""
    with chunk.fmt():
        if device:
            out = torch.empty(lib().dq_wire_bytes(*chunk.runs), dtype=torch.uint8, device=chunk.data.device)
            check(lib().dq_serialize_chunk(_ptr(chunk.data), chunk.chunk_index, *chunk.runs,
                                           _ptr(out), _stream()))
            return out
        soa = chunk.data.cpu().numpy()
        out = np.zeros(lib().dq_wire_bytes(*chunk.runs), np.uint8)
        check(lib().dq_to_reference_wire(soa.ctypes.data_as(C.c_void_p), chunk.chunk_index, *chunk.runs,
                                         out.ctypes.data_as(C.c_void_p)))
        return out.tobytes()


def soa_from_reference(buf: bytes, cfg: Optional[CodecConfig] = None):
    """Strict parse of reference wire bytes into the device layout (host numpy array)
    -> (chunk_index, n8, n4, n2, n16, soa)."""
    b = np.frombuffer(buf, np.uint8).copy()
    count = int(np.frombuffer(b[4:8].tobytes(), np.uint32)[0]) if b.size >= 8 else 0
    cap = max(len(buf) + 64 * min(count, len(buf)), 1)  # passthrough records carry no scales on the wire
    soa = np.zeros(cap, np.uint8)
    ci, n8, n4, n2, n16 = (C.c_uint32() for _ in range(5))
    with _fmt_of(cfg):
        check(lib().dq_from_reference_wire(b.ctypes.data_as(C.c_void_p), b.size, soa.ctypes.data_as(C.c_void_p),
                                           soa.size, C.byref(ci), C.byref(n8), C.byref(n4), C.byref(n2),
                                           C.byref(n16)))
    runs = (n8.value, n4.value, n2.value, n16.value)
    return (ci.value,) + runs + (soa[: chunk_bytes(*runs, cfg=cfg)],)


def parse_chunk(buf, device="cuda", cfg: Optional[CodecConfig] = None) -> DeviceChunk:
    """proj/src/codec.cpp:345-399 — raises MalformedBuffer on any malformed buffer.

    ``buf``: host bytes (parsed on the host), or a CUDA uint8 tensor (parsed and
    validated on the GPU by dq_parse_chunk); ``cfg``: the scale format (default s=16,
    hierarchical), like the reference's CodecConfig argument."""
    gs, hier = (16, True) if cfg is None else (cfg.group_size, cfg.hierarchical_scales)
    if isinstance(buf, torch.Tensor):
        if not (buf.is_cuda and buf.dtype == torch.uint8 and buf.is_contiguous()):
            raise InvalidArgument(2, "device wire buffer must be a contiguous CUDA uint8 tensor")
        ci, n8, n4, n2, n16 = (C.c_uint32() for _ in range(5))
        outs = (C.byref(ci), C.byref(n8), C.byref(n4), C.byref(n2), C.byref(n16))
        # validate and read the run lengths, then parse into a buffer of the device size
        with _fmt_of(cfg):
            check(lib().dq_parse_chunk(_ptr(buf), buf.numel(), None, 0, *outs, _stream()))
            runs = (n8.value, n4.value, n2.value, n16.value)
            data = torch.empty(max(lib().dq_chunk_bytes(*runs), 1), dtype=torch.uint8, device=buf.device)
            check(lib().dq_parse_chunk(_ptr(buf), buf.numel(), _ptr(data), data.numel(), *outs, _stream()))
        return DeviceChunk(ci.value, n8.value, n4.value, n2.value, data, n16.value, gs, hier)
    ci, n8, n4, n2, n16, soa = soa_from_reference(buf, cfg)
    data = torch.from_numpy(soa.copy() if soa.size else np.zeros(1, np.uint8)).to(device)
    return DeviceChunk(ci, n8, n4, n2, data, n16, gs, hier)


def compute_stats(x: torch.Tensor):
    """proj/src/stats.cpp:23-35 -> (mean, sq_norm) float32 tensors, one per super-group."""
    x = _f32(x, x.numel(), "gradient")
    T = (x.numel() + 255) // 256
    mean = torch.empty(T, dtype=torch.float32, device=x.device)
    sq = torch.empty_like(mean)
    check(lib().dq_compute_stats(_ptr(x), x.numel(), _ptr(mean), _ptr(sq), _stream()))
    return mean, sq


def reduce_stats(means: torch.Tensor, sqs: torch.Tensor):
    """proj/src/stats.cpp:37-54: rank-ordered fp64 reduction of [n_workers, n_sg] stats."""
    means, sqs = means.contiguous(), sqs.contiguous()
    n, T = means.shape
    gm = torch.empty(T, dtype=torch.float32, device=means.device)
    gs = torch.empty_like(gm)
    check(lib().dq_reduce_stats(_ptr(means), _ptr(sqs), n, T, _ptr(gm), _ptr(gs), _stream()))
    return gm, gs


@dataclass
class BitAllocation:
    """proj/include/dynamiq/allocation.hpp:40-45"""
    widths: torch.Tensor       # uint8 per super-group (original order)
    permutation: torch.Tensor  # int32: position k holds super-group permutation[k]
    payload_bits: int
    u: float
    counts: tuple              # (n8, n4, n2)


class Context:
    """One device context (scratch owner); mirrors one worker's engine state."""

    def __init__(self, config: Optional[PipelineConfig] = None, device: Optional[int] = None):
        self.config = config or PipelineConfig()
        self.device = torch.cuda.current_device() if device is None else device
        h = C.c_void_p()
        cfg = self.config._c()
        check(lib().dq_ctx_create(C.byref(cfg), self.device, C.byref(h)))
        self.h = h

    def set_config(self, config: PipelineConfig) -> None:
        cfg = config._c()
        check(lib().dq_ctx_set_config(self.h, C.byref(cfg)))
        self.config = config

    def profile(self, on: bool = True) -> None:
        check(lib().dq_profile_enable(self.h, int(on)))

    def read_profile(self, reset: bool = True) -> dict:
        """{family: {"launches", "ms", "bytes"}} accumulated since the last reset."""
        arr = (_lib.KernelProfile * 16)()
        n = C.c_int()
        check(lib().dq_profile_read(self.h, arr, 16, C.byref(n), int(reset)))
        return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].ms, "bytes": arr[i].bytes}
                for i in range(min(n.value, 16))}

    def wait(self) -> dict:
        """Wait for this context's last round and return its full info (allocation,
        accounting, device time) - what an asynchronous round leaves unfilled."""
        info = RoundInfo()
        check(lib().dq_round_wait(self.h, C.byref(info)))
        return _info_dict(info)

    def host_allocations(self) -> dict:
        """Diagnostics: rounds whose bit allocation the host finished ("finished", rare) and
        rounds that only asked the host for the candidates' glibc thresholds ("consulted")."""
        f, c = C.c_uint64(), C.c_uint64()
        check(lib().dq_ctx_host_allocations(self.h, C.byref(f), C.byref(c)))
        return {"finished": f.value, "consulted": c.value}

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().dq_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict = {}


def _ctx_for(config: PipelineConfig) -> Context:
    dev = torch.cuda.current_device()
    c = _default_ctx.get(dev)
    if c is None:
        c = _default_ctx[dev] = Context(config, dev)
    else:
        c.set_config(config)
    return c


def allocate_fast(sq_norms: torch.Tensor, budget_bits: float, ctx: Optional[Context] = None) -> BitAllocation:
    """proj/src/allocation.cpp:228-260 + build_permutation (W = {2,4,8}, s=16, S=256)."""
    ctx = ctx or _ctx_for(PipelineConfig())
    F = _f32(sq_norms, sq_norms.numel(), "sq_norms")
    T = F.numel()
    widths = torch.empty(max(T, 1), dtype=torch.uint8, device=F.device)
    perm = torch.empty(max(T, 1), dtype=torch.int32, device=F.device)
    u, pay = C.c_double(), C.c_uint64()
    counts = (C.c_uint32 * 3)()
    check(lib().dq_allocate_fast(ctx.h, _ptr(F), T, float(budget_bits), _ptr(widths), _ptr(perm), C.byref(u),
                                 C.byref(pay), counts, _stream()))
    return BitAllocation(widths[:T], perm[:T], pay.value, u.value, tuple(counts))


def allocate_general(sq_norms: torch.Tensor, budget_bits: float, ctx: Optional[Context] = None) -> BitAllocation:
    """proj/src/allocation.cpp:121-168 (W = {2,4,8}, the set run_round uses) + build_permutation;
    ``u`` is the resolved base threshold."""
    ctx = ctx or _ctx_for(PipelineConfig())
    F = _f32(sq_norms, sq_norms.numel(), "sq_norms")
    T = F.numel()
    widths = torch.empty(max(T, 1), dtype=torch.uint8, device=F.device)
    perm = torch.empty(max(T, 1), dtype=torch.int32, device=F.device)
    u, pay = C.c_double(), C.c_uint64()
    counts = (C.c_uint32 * 3)()
    check(lib().dq_allocate_general(ctx.h, _ptr(F), T, float(budget_bits), _ptr(widths), _ptr(perm), C.byref(u),
                                    C.byref(pay), counts, _stream()))
    return BitAllocation(widths[:T], perm[:T], pay.value, u.value, tuple(counts))


@dataclass
class FastAllocatorState:
    """proj/include/dynamiq/allocation.hpp:75-79"""
    lo: float = -1e6
    hi: float = 1e6
    u: float = 0.0


def allocate_fast_stateful(sq_norms: torch.Tensor, budget_bits: float, state: FastAllocatorState,
                           ctx: Optional[Context] = None) -> BitAllocation:
    """proj/src/allocation.cpp:262-300: widths at the carried ``state.u`` (projected to the
    largest in-budget plateau when over budget); ``state`` takes one bisection step."""
    ctx = ctx or _ctx_for(PipelineConfig())
    F = _f32(sq_norms, sq_norms.numel(), "sq_norms")
    T = F.numel()
    widths = torch.empty(max(T, 1), dtype=torch.uint8, device=F.device)
    perm = torch.empty(max(T, 1), dtype=torch.int32, device=F.device)
    st = (C.c_double * 3)(state.lo, state.hi, state.u)
    u, pay = C.c_double(), C.c_uint64()
    counts = (C.c_uint32 * 3)()
    check(lib().dq_allocate_fast_stateful(ctx.h, _ptr(F), T, float(budget_bits), st, _ptr(widths), _ptr(perm),
                                          C.byref(u), C.byref(pay), counts, _stream()))
    state.lo, state.hi, state.u = st[0], st[1], st[2]
    return BitAllocation(widths[:T], perm[:T], pay.value, u.value, tuple(counts))


def ablation_ladder(base: PipelineConfig) -> list:
    """proj/src/engine.cpp:420-450: the Table-6 ladder of configs, each rung adding one
    ingredient: uniform -> non_uniform -> variable_width -> hierarchical -> correlated."""
    from dataclasses import replace
    uniform = replace(base, non_uniform=False, variable_width=False, allocator=KIND_FIXED, fixed_width=4,
                      hierarchical_scales=False, correlated=False, group_size=32)
    non_uniform = replace(uniform, non_uniform=True)
    variable = replace(non_uniform, variable_width=True,
                       allocator=KIND_FAST if base.allocator == KIND_FIXED else base.allocator)
    hierarchical = replace(variable, hierarchical_scales=True, group_size=16)
    correlated = replace(hierarchical, correlated=True)
    return [("uniform", uniform), ("non_uniform", non_uniform), ("variable_width", variable),
            ("hierarchical", hierarchical), ("correlated", correlated)]


@dataclass
class RoundResult:
    """proj/include/dynamiq/engine.hpp:45-54 (exact fp64 sum not materialized)."""
    synced: torch.Tensor
    vnmse: float
    mse: float
    wire_hash: int
    u: float
    payload_bits: int
    info: dict
    widths: Optional[np.ndarray] = None
    permutation: Optional[np.ndarray] = None


def _info_dict(info: RoundInfo) -> dict:
    return {k: getattr(info, k) for k, _ in RoundInfo._fields_}


def run_round(worker_values: Sequence[torch.Tensor], config: PipelineConfig, collect_wire: bool = False,
              with_allocation: bool = False, out: Optional[torch.Tensor] = None,
              ctx: Optional[Context] = None, metrics: bool = True) -> RoundResult:
    """One full round with every worker's gradient on this GPU (simulated hops).

    Same inputs/outputs as the reference's run_round (proj/src/engine.cpp:269-418);
    ``collect_wire`` also computes the reference's wire_hash over the serialized
    messages (slow; for parity tests)."""
    if len(worker_values) == 0:
        raise InvalidArgument(2, "no workers")
    if len(worker_values) != config.n_workers:
        raise InvalidArgument(2, "worker count does not match config")
    d = worker_values[0].numel()
    if d == 0:
        raise InvalidArgument(2, "empty gradient")
    xs = [_f32(w, d, "worker gradient") if w.numel() == d else None for w in worker_values]
    if any(x is None for x in xs):
        raise InvalidArgument(2, "worker gradients must have equal length")
    ctx = ctx or _ctx_for(config)
    if ctx.config is not config:
        ctx.set_config(config)
    if out is None:
        out = torch.empty(d, dtype=torch.float32, device=xs[0].device)
    ptrs = (C.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
    info = RoundInfo()
    flags = (1 if collect_wire else 0) | (0 if metrics else 2)
    check(lib().dq_sim_round(ctx.h, ptrs, d, _ptr(out), flags, C.byref(info), _stream()))
    res = RoundResult(out, info.vnmse, info.mse, info.wire_hash, info.u, info.payload_bits, _info_dict(info))
    if with_allocation and config.n_workers > 1:
        T = (d + 255) // 256
        w = np.zeros(T, np.uint8)
        p = np.zeros(T, np.uint32)
        check(lib().dq_round_allocation(ctx.h, w.ctypes.data_as(C.POINTER(C.c_uint8)),
                                        p.ctypes.data_as(C.POINTER(C.c_uint32)), T))
        res.widths, res.permutation = w, p
    return res


def run_round_host(worker_values: Sequence[np.ndarray], config: PipelineConfig,
                   ctx: Optional[Context] = None) -> tuple:
    """run_round on HOST buffers (the e2e path: H2D of every input and D2H of the sum inside)."""
    ctx = ctx or _ctx_for(config)
    if ctx.config is not config:
        ctx.set_config(config)
    xs = [np.ascontiguousarray(w, np.float32) for w in worker_values]
    d = xs[0].size
    out = np.empty(d, np.float32)
    ptrs = (C.c_void_p * len(xs))(*[x.ctypes.data for x in xs])
    info = RoundInfo()
    check(lib().dq_run_round_host(ctx.h, ptrs, d, out.ctypes.data_as(C.c_void_p), C.byref(info), _stream()))
    return out, _info_dict(info)


class Event(C.Structure):
    _fields_ = [("sender", C.c_uint32), ("receiver", C.c_uint32), ("slot", C.c_uint32), ("stage", C.c_uint32)]


def schedule(n_workers: int, topology: int, chunk: int) -> dict:
    """proj/include/dynamiq/topology.hpp ChunkPlan of `chunk`: reduce events (sender, receiver,
    hop slot, executor stage), sink compression slot, slot count, gather message count."""
    ev = (Event * 512)()
    ne, ss, ns, ng = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib().dq_schedule(n_workers, topology, chunk, ev, 512, C.byref(ne), C.byref(ss), C.byref(ns), C.byref(ng)))
    return {"events": [(ev[i].sender, ev[i].receiver, ev[i].slot, ev[i].stage) for i in range(ne.value)],
            "sink_slot": ss.value, "n_slots": ns.value, "n_gather": ng.value}


TRANSPORT_PEER, TRANSPORT_NCCL = 0, 1


class Communicator:
    """Distributed all-reduce: one process per GPU.

    Ring transport ``"peer"`` (default): the fused hop kernels store compressed
    units straight into the neighbour's HBM over NVLink (CUDA IPC, per-unit flags);
    ``"nccl"``: NCCL point-to-point between the fused kernels.  ``torch.distributed``
    (any backend) only ships the 128-byte NCCL id."""

    def __init__(self, config: PipelineConfig, rank: int, world_size: int, group=None,
                 transport: Optional[str] = None):
        import torch.distributed as dist
        if config.n_workers != world_size:
            raise InvalidArgument(2, "config.n_workers must equal the world size")
        self.ctx = Context(config)
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            check(lib().dq_comm_unique_id(uid.ctypes.data_as(C.POINTER(C.c_uint8))))
        obj = [uid.tobytes()]
        # src is a global rank: the group's rank 0 (a subgroup need not contain rank 0)
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = np.frombuffer(obj[0], np.uint8).copy()
        check(lib().dq_comm_init(self.ctx.h, rank, world_size, uid.ctypes.data_as(C.POINTER(C.c_uint8))))
        if transport is not None:
            if transport not in ("peer", "nccl"):
                raise InvalidArgument(2, f"unknown transport {transport!r}")
            check(lib().dq_comm_set_transport(self.ctx.h, TRANSPORT_PEER if transport == "peer" else TRANSPORT_NCCL))
        self.rank, self.world_size = rank, world_size

    @property
    def transport(self) -> str:
        """Active ring transport ("peer" or "nccl"; peer falls back to nccl if mapping fails)."""
        t = C.c_int()
        check(lib().dq_comm_get_transport(self.ctx.h, C.byref(t)))
        return "peer" if t.value == TRANSPORT_PEER else "nccl"

    def allreduce(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, async_op: bool = False):
        """SUM estimate of every rank's ``x`` (caller divides by n for a mean).

        ``async_op=False``: waits for the round, returns ``(out, info)``.  ``async_op=True``:
        enqueues the round on the current stream without any host synchronisation (it can be
        captured in a CUDA graph) and returns ``out``; ``self.ctx.wait()`` gives the info."""
        x = _f32(x, x.numel(), "gradient")
        if out is None:
            out = torch.empty_like(x)
        if async_op:
            check(lib().dq_allreduce(self.ctx.h, _ptr(x), _ptr(out), x.numel(), None, _stream()))
            return out
        info = RoundInfo()
        check(lib().dq_allreduce(self.ctx.h, _ptr(x), _ptr(out), x.numel(), C.byref(info), _stream()))
        return out, _info_dict(info)
