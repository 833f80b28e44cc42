"""CPU checks of the C-ABI library (no GPU needed).

* libdynamiq_b200.so loads and exports every entry point include/dynamiq_b200.h declares;
* config defaults equal the reference's PipelineConfig defaults (engine.hpp:22-43);
* the host-side wire converters are exact inverses on reference bytes made by the oracle,
  and the strict parser rejects malformed buffers like parse_chunk (codec.cpp:345-399,
  proj/tests/test_codec.cpp:180-223);
* calls needing a device fail loudly (status code), never fall back to the CPU.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from tests.golden.make_golden import det_values

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2602_08923_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dynamiq_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dq_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    from paper_2602_08923_b200._lib import SIGNATURES
    syms = declared_symbols()
    assert len(syms) >= 24
    for s in syms:
        assert hasattr(L, s), s
        assert s in SIGNATURES, f"{s} missing from the ctypes signature table"


def test_no_unresolved_internal_symbols():
    """Every dq:: symbol the library references is defined in it (RTLD_NOW load in lib())."""
    import subprocess
    from paper_2602_08923_b200 import _lib
    out = subprocess.run(["nm", "-D", "--undefined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "_ZN2dq" not in out, out


def test_version_and_defaults(L):
    from paper_2602_08923_b200._lib import Config
    assert L.dq_version() >= 1
    c = Config()
    L.dq_config_default(C.byref(c))
    assert (c.n_workers, c.group_size, c.super_group_size, c.budget_bits) == (4, 16, 256, 5.0)
    assert (c.non_uniform, c.variable_width, c.hierarchical_scales, c.correlated) == (1, 1, 1, 1)
    assert (c.fixed_width, c.allocator, c.topology, c.codec, c.seed, c.round, c.threads) == (4, 1, 0, 0, 1, 0, 1)


def _widths(runs):
    runs = tuple(runs) + (0,) * (4 - len(runs))
    return [8] * runs[0] + [4] * runs[1] + [2] * runs[2] + [16] * runs[3]


@pytest.mark.parametrize("runs", [(0, 0, 0, 0), (1, 0, 0, 0), (3, 5, 9, 0), (64, 0, 1, 0), (70, 70, 70, 0),
                                  (0, 0, 0, 1), (2, 3, 4, 5), (64, 0, 0, 64)])
def test_chunk_bytes_match_wire_size(L, port, runs):
    w = _widths(runs)
    assert L.dq_wire_bytes(*runs) * 8 == port.compressed_size_bits(w)
    assert L.dq_chunk_bytes(*runs) == L.dq_wire_bytes(*runs) - 24 + 18 * runs[3]


def _ref_bytes(port, runs, seed=1):
    w = np.array(_widths(runs), np.uint8)
    v = det_values(seed, w.size * 256)
    return port.compress_chunk(v, w, port.codec(), port.qctx(seed, 0, 3, 1, 4, True), first_sg=2)


@pytest.mark.parametrize("runs", [(1, 0, 0, 0), (0, 1, 0, 0), (0, 0, 1, 0), (3, 5, 9, 0), (65, 2, 64, 0),
                                  (0, 130, 1, 0), (0, 0, 0, 1), (1, 2, 3, 4), (70, 0, 0, 70)])
def test_wire_roundtrip(port, runs):
    import paper_2602_08923_b200 as dq
    ref = _ref_bytes(port, runs)
    ci, n8, n4, n2, n16, soa = dq.soa_from_reference(ref)
    assert (ci, n8, n4, n2, n16) == (3,) + runs
    out = np.zeros(len(ref), np.uint8)
    from paper_2602_08923_b200._lib import check, lib
    check(lib().dq_to_reference_wire(soa.ctypes.data_as(C.c_void_p), ci, n8, n4, n2, n16,
                                     out.ctypes.data_as(C.c_void_p)))
    assert out.tobytes() == ref


def test_malformed_rejected(port):
    import paper_2602_08923_b200 as dq
    ref = _ref_bytes(port, (0, 1, 1), seed=9)
    for cut in (1, len(ref) // 2, len(ref) - 1):
        with pytest.raises(dq.MalformedBuffer):
            dq.soa_from_reference(ref[:cut])
    with pytest.raises(dq.MalformedBuffer):
        dq.soa_from_reference(ref + b"\0")
    t = bytearray(ref)
    t[8] += 1
    with pytest.raises(dq.MalformedBuffer):
        dq.soa_from_reference(bytes(t))
    zeros = port.compress_chunk(np.zeros(512, np.float32), np.array([4, 2], np.uint8), port.codec(), port.qctx(9))
    z = bytearray(zeros)
    z[-1] = 0xFF
    with pytest.raises(dq.MalformedBuffer):
        dq.soa_from_reference(bytes(z))
    # passthrough records: their own truncation message, no zero-scale rule (codec.cpp:371-376)
    p16 = _ref_bytes(port, (1, 0, 0, 2), seed=5)
    with pytest.raises(dq.MalformedBuffer, match="truncated width-16 body"):
        dq.soa_from_reference(p16[:-1])
    with pytest.raises(dq.MalformedBuffer, match="truncated super-group body"):
        dq.soa_from_reference(p16[:24 + 100])


def test_random_flips_reject_or_roundtrip(port):
    """proj/tests/test_codec.cpp:209-222: a flipped bit is rejected or re-serializes identically."""
    import paper_2602_08923_b200 as dq
    from paper_2602_08923_b200._lib import check, lib
    ref = _ref_bytes(port, (1, 1, 1, 1), seed=4)
    rng = np.random.default_rng(0)
    for _ in range(400):
        t = bytearray(ref)
        pos = int(rng.integers(0, len(t)))
        t[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            ci, n8, n4, n2, n16, soa = dq.soa_from_reference(bytes(t))
        except (dq.MalformedBuffer, dq.InvalidArgument):
            continue
        out = np.zeros(dq.wire_bytes(n8, n4, n2, n16), np.uint8)
        check(lib().dq_to_reference_wire(soa.ctypes.data_as(C.c_void_p), ci, n8, n4, n2, n16,
                                         out.ctypes.data_as(C.c_void_p)))
        assert out.tobytes() == bytes(t)


def test_device_calls_fail_loudly_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2602_08923_b200._lib import Config
    c = Config()
    L.dq_config_default(C.byref(c))
    h = C.c_void_p()
    rc = L.dq_ctx_create(C.byref(c), 0, C.byref(h))
    assert rc == 5 and b"cuda" in L.dq_last_error().lower()


def test_invalid_config_rejected(L):
    from paper_2602_08923_b200._lib import Config
    c = Config()
    L.dq_config_default(C.byref(c))
    c.topology = 1
    c.n_workers = 3  # butterfly needs a power of two (engine.cpp:248-249)
    h = C.c_void_p()
    assert L.dq_ctx_create(C.byref(c), 0, C.byref(h)) == 2
    L.dq_config_default(C.byref(c))
    c.group_size = 12  # not a power of two in 8..128 (the device codec's group sizes)
    assert L.dq_ctx_create(C.byref(c), 0, C.byref(h)) == 2
    L.dq_config_default(C.byref(c))
    c.super_group_size = 512
    assert L.dq_ctx_create(C.byref(c), 0, C.byref(h)) == 2
