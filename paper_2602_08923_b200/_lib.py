"""Loader for the native library ``libdynamiq_b200.so`` (C-ABI: include/dynamiq_b200.h).

There is no fallback: if the library is missing or fails to load, every entry
point raises.  ``build()`` compiles it in-tree with nvcc for sm_100a.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdynamiq_b200.so")
if os.environ.get("DQ_LIB_VARIANT"):  # experiments: an in-tree build variant (variants/<name>.so)
    LIB_PATH = os.path.join(HERE, "variants", os.environ["DQ_LIB_VARIANT"] + ".so")

DQ_OK, DQ_EINVAL, DQ_EINFEASIBLE, DQ_EMALFORMED, DQ_ECUDA, DQ_ENCCL = 0, 2, 3, 4, 5, 6


class DqError(RuntimeError):
    """Base class; ``code`` is the dq_status returned by the C-ABI."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(DqError, ValueError):
    """std::invalid_argument in the reference (CLI exit code 2)."""


class InfeasibleBudget(DqError):
    """dynamiq::InfeasibleBudget (proj/include/dynamiq/allocation.hpp:14-16; CLI exit 3)."""


class MalformedBuffer(DqError):
    """std::runtime_error("malformed compressed buffer: ...") (proj/src/codec.cpp:20-22)."""


class CudaError(DqError):
    pass


class NcclError(DqError):
    pass


_EXC = {DQ_EINVAL: InvalidArgument, DQ_EINFEASIBLE: InfeasibleBudget, DQ_EMALFORMED: MalformedBuffer,
        DQ_ECUDA: CudaError, DQ_ENCCL: NcclError}


class Config(C.Structure):
    _fields_ = [("n_workers", C.c_uint32), ("group_size", C.c_uint32), ("super_group_size", C.c_uint32),
                ("budget_bits", C.c_double), ("non_uniform", C.c_int32), ("variable_width", C.c_int32),
                ("hierarchical_scales", C.c_int32), ("correlated", C.c_int32), ("fixed_width", C.c_int32),
                ("allocator", C.c_int32), ("topology", C.c_int32), ("codec", C.c_int32),
                ("seed", C.c_uint64), ("round", C.c_uint64), ("threads", C.c_uint32)]


class QCtx(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("round", C.c_uint64), ("chunk_index", C.c_uint32),
                ("hop_slot", C.c_uint32), ("n_slots", C.c_uint32), ("correlated", C.c_int32)]


class RoundInfo(C.Structure):
    _fields_ = [("wire_hash", C.c_uint64), ("vnmse", C.c_double), ("mse", C.c_double), ("u", C.c_double),
                ("payload_bits", C.c_uint64), ("stats_bits", C.c_uint64), ("wire_payload_bits", C.c_uint64),
                ("scale_bits", C.c_uint64), ("header_bits", C.c_uint64), ("repr_bits", C.c_uint64),
                ("compressed_coordinates", C.c_uint64), ("transmitted_coordinates", C.c_uint64),
                ("n8", C.c_uint32), ("n4", C.c_uint32), ("n2", C.c_uint32), ("alloc_passes", C.c_uint32),
                ("ms_total", C.c_double)]


class KernelProfile(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("ms", C.c_double), ("bytes", C.c_double)]


# every symbol declared in include/dynamiq_b200.h: name -> (restype, argtypes)
_P, _V, _u8p, _u32p = C.POINTER, C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32)
_fp = C.POINTER(C.c_float)
SIGNATURES = {
    "dq_version": (C.c_int, []),
    "dq_build_flags": (C.c_int, []),
    "dq_last_error": (C.c_char_p, []),
    "dq_config_default": (None, [_P(Config)]),
    "dq_ctx_create": (C.c_int, [_P(Config), C.c_int, _P(_V)]),
    "dq_ctx_destroy": (C.c_int, [_V]),
    "dq_ctx_set_config": (C.c_int, [_V, _P(Config)]),
    "dq_chunk_bytes": (C.c_size_t, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "dq_wire_bytes": (C.c_size_t, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "dq_compress_chunk": (C.c_int, [_V, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _P(QCtx), C.c_uint32, C.c_int,
                                    _V, _V]),
    "dq_dar_chunk": (C.c_int, [_V, _V, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _P(QCtx), C.c_uint32, C.c_int,
                               _V, _V]),
    "dq_da_chunk": (C.c_int, [_V, _V, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _V]),
    "dq_decompress_chunk": (C.c_int, [_V, _V, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _V]),
    "dq_to_reference_wire": (C.c_int, [_V, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _V]),
    "dq_from_reference_wire": (C.c_int, [_V, C.c_size_t, _V, C.c_size_t, _u32p, _u32p, _u32p, _u32p, _u32p]),
    "dq_serialize_chunk": (C.c_int, [_V, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _V, _V]),
    "dq_parse_chunk": (C.c_int, [_V, C.c_size_t, _V, C.c_size_t, _P(C.c_uint32), _P(C.c_uint32),
                                 _P(C.c_uint32), _P(C.c_uint32), _P(C.c_uint32), _V]),
    "dq_compute_stats": (C.c_int, [_V, C.c_size_t, _V, _V, _V]),
    "dq_reduce_stats": (C.c_int, [_V, _V, C.c_uint32, C.c_size_t, _V, _V, _V]),
    "dq_allocate_fast": (C.c_int, [_V, _V, C.c_size_t, C.c_double, _V, _V, _P(C.c_double), _P(C.c_uint64),
                                   _u32p, _V]),
    "dq_allocate_general": (C.c_int, [_V, _V, C.c_size_t, C.c_double, _V, _V, _P(C.c_double), _P(C.c_uint64),
                                      _P(C.c_uint32), _V]),
    "dq_allocate_fast_stateful": (C.c_int, [_V, _V, C.c_size_t, C.c_double, _P(C.c_double), _V, _V,
                                            _P(C.c_double), _P(C.c_uint64), _P(C.c_uint32), _V]),
    "dq_sim_round": (C.c_int, [_V, _P(_V), C.c_size_t, _V, C.c_int, _P(RoundInfo), _V]),
    "dq_run_round_host": (C.c_int, [_V, _P(_V), C.c_size_t, _V, _P(RoundInfo), _V]),
    "dq_round_allocation": (C.c_int, [_V, _u8p, _u32p, C.c_size_t]),
    "dq_selftest": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, _P(C.c_uint64)]),
    "dq_profile_enable": (C.c_int, [_V, C.c_int]),
    "dq_profile_read": (C.c_int, [_V, _P(KernelProfile), C.c_int, _P(C.c_int), C.c_int]),
    "dq_schedule": (C.c_int, [C.c_uint32, C.c_int, C.c_uint32, _V, C.c_uint32, _P(C.c_uint32), _P(C.c_uint32),
                              _P(C.c_uint32), _P(C.c_uint32)]),
    "dq_comm_unique_id": (C.c_int, [_u8p]),
    "dq_comm_init": (C.c_int, [_V, C.c_int, C.c_int, _u8p]),
    "dq_allreduce": (C.c_int, [_V, _V, _V, C.c_size_t, _P(RoundInfo), _V]),
    "dq_round_wait": (C.c_int, [_V, _P(RoundInfo)]),
    "dq_codec_format_set": (C.c_int, [C.c_uint32, C.c_int, _P(C.c_uint32), _P(C.c_int)]),
    "dq_debug_force_host_alloc": (C.c_int, [C.c_int]),
    "dq_ctx_host_allocations": (C.c_int, [_V, _P(C.c_uint64), _P(C.c_uint64)]),
    "dq_comm_set_transport": (C.c_int, [_V, C.c_int]),
    "dq_comm_get_transport": (C.c_int, [_V, _P(C.c_int)]),
}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile the CUDA/C++ sources (sm_100a) into LIB_PATH."""
    out = subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc"), "-j4"], capture_output=not verbose,
                         text=True)
    if out.returncode != 0:
        raise RuntimeError("building libdynamiq_b200.so failed:\n" + (out.stdout or "") + (out.stderr or ""))
    return LIB_PATH


def lib() -> C.CDLL:
    """The loaded native library (raises if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run paper_2602_08923_b200._lib.build()")
        L = C.CDLL(LIB_PATH, mode=os.RTLD_NOW)  # resolve every symbol now: a broken build fails here
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != DQ_OK:
        msg = lib().dq_last_error().decode(errors="replace")
        raise _EXC.get(rc, DqError)(rc, msg)
