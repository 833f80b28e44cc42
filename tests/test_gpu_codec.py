"""Parity of the sm_100a codec kernels with the oracle: bit-exact wire bytes.

Mirrors the reference's codec tests (proj/tests/test_codec.cpp) but compares
the device output byte for byte with the CPU oracle on the same inputs.
"""
import zlib

import numpy as np
import pytest

from tests.util import sg_block, sorted_widths

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_08923_b200 as dq
    return dq


RUNS = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (3, 5, 9), (70, 1, 60), (0, 130, 0), (64, 64, 64),
        (0, 0, 0, 1), (2, 3, 4, 5), (64, 0, 1, 70)]  # width-16 passthrough runs last (codec.cpp:82-86)
SLOTS = [(1, 0), (2, 0), (2, 1), (3, 2), (4, 0), (4, 1), (4, 3), (5, 4), (6, 2), (7, 6), (8, 0), (8, 1),
         (8, 4), (8, 7), (16, 0), (16, 9)]


def _codec(ora, non_uniform=True):
    return ora.codec(16, 256, True, non_uniform)


@pytest.mark.parametrize("runs", RUNS)
@pytest.mark.parametrize("kind", ["mixed", "lognormal"])
def test_compress_bytes_match(dq, port, runs, kind):
    rng = np.random.default_rng(zlib.crc32(repr((runs, kind)).encode()))
    w = sorted_widths(*runs)
    v = sg_block(rng, len(w), kind)
    for n_slots, slot in [(1, 0), (4, 2), (8, 7)]:
        for corr in (True, False):
            q = dq.QuantContext(dq.SharedSeed(7, 3), chunk_index=5, hop_slot=slot, n_slots=n_slots, correlated=corr)
            got = dq.serialize_chunk(dq.compress_chunk(torch.from_numpy(v).cuda(), w, dq.CodecConfig(), q, 11))
            want = port.compress_chunk(v, w, _codec(port), port.qctx(7, 3, 5, slot, n_slots, corr), first_sg=11)
            assert got == want, (runs, kind, n_slots, slot, corr)


@pytest.mark.parametrize("n_slots,slot", SLOTS)
def test_compress_all_slot_counts(dq, port, n_slots, slot):
    rng = np.random.default_rng(n_slots * 100 + slot)
    w = sorted_widths(20, 20, 24)
    v = sg_block(rng, len(w), "normal")
    q = dq.QuantContext(dq.SharedSeed(1, 0), chunk_index=2, hop_slot=slot, n_slots=n_slots)
    got = dq.serialize_chunk(dq.compress_chunk(torch.from_numpy(v).cuda(), w, dq.CodecConfig(), q, 1000))
    want = port.compress_chunk(v, w, _codec(port), port.qctx(1, 0, 2, slot, n_slots, True), first_sg=1000)
    assert got == want


@pytest.mark.parametrize("non_uniform", [True, False])
def test_uniform_codebooks(dq, port, non_uniform):
    rng = np.random.default_rng(5)
    w = sorted_widths(10, 10, 10)
    v = sg_block(rng, len(w), "mixed")
    cfg = dq.CodecConfig(non_uniform=non_uniform)
    q = dq.QuantContext(dq.SharedSeed(3, 1), chunk_index=0, hop_slot=1, n_slots=4)
    got = dq.serialize_chunk(dq.compress_chunk(torch.from_numpy(v).cuda(), w, cfg, q, 0))
    want = port.compress_chunk(v, w, _codec(port, non_uniform), port.qctx(3, 1, 0, 1, 4, True))
    assert got == want


@pytest.mark.parametrize("runs", RUNS)
def test_dar_bytes_match(dq, port, runs):
    """Fused decompress-accumulate-recompress == reference DAR (codec.cpp:238-266)."""
    rng = np.random.default_rng(sum(runs))
    w = sorted_widths(*runs)
    base = sg_block(rng, len(w), "lognormal")
    local = sg_block(rng, len(w), "mixed")
    cc = _codec(port)
    for n_slots, slot in [(4, 1), (8, 3), (8, 7), (2, 1), (3, 1)]:
        inc = port.compress_chunk(base, w, cc, port.qctx(9, 0, 1, slot - 1, n_slots, True), first_sg=3)
        want = port.dar_chunk(inc, local, cc, port.qctx(9, 0, 1, slot, n_slots, True), first_sg=3)
        chunk = dq.parse_chunk(inc)
        q = dq.QuantContext(dq.SharedSeed(9, 0), chunk_index=1, hop_slot=slot, n_slots=n_slots)
        got = dq.serialize_chunk(dq.decompress_accumulate_recompress(chunk, torch.from_numpy(local).cuda(),
                                                                     dq.CodecConfig(), q, 3))
        assert got == want, (runs, n_slots, slot)


def test_fused_equals_unfused(dq):
    """proj/tests/test_codec.cpp:118-140 on the device path."""
    rng = np.random.default_rng(11)
    w = sorted_widths(1, 2, 1)
    cfg = dq.CodecConfig()
    for trial in range(20):
        base = torch.from_numpy(sg_block(rng, 4, "normal") * 3).cuda()
        local = torch.from_numpy(sg_block(rng, 4, "normal")).cuda()
        inc = dq.compress_chunk(base, w, cfg, dq.QuantContext(dq.SharedSeed(trial), 0, 0, 4))
        hop = dq.QuantContext(dq.SharedSeed(trial), 0, 1, 4)
        fused = dq.decompress_accumulate_recompress(inc, local, cfg, hop)
        dec = dq.decompress_chunk(inc, cfg) + local
        unfused = dq.compress_chunk(dec, w, cfg, hop)
        assert torch.equal(fused.data, unfused.data)


@pytest.mark.parametrize("runs", RUNS)
def test_decompress_and_da_match(dq, port, runs):
    rng = np.random.default_rng(77 + sum(runs))
    w = sorted_widths(*runs)
    v = sg_block(rng, len(w), "mixed")
    cc = _codec(port)
    buf = port.compress_chunk(v, w, cc, port.qctx(4, 0, 0, 0, 4, True))
    chunk = dq.parse_chunk(buf)
    got = dq.decompress_chunk(chunk, dq.CodecConfig()).cpu().numpy()
    want = port.decompress_chunk(buf, cc, v.size)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    acc = sg_block(rng, len(w), "normal")
    acc_t = torch.from_numpy(acc).cuda()
    dq.decompress_accumulate(chunk, acc_t, dq.CodecConfig())
    want2 = port.decompress_accumulate(buf, cc, acc)
    assert np.array_equal(acc_t.cpu().numpy().view(np.uint32), want2.view(np.uint32))


def test_sg_known_answer(dq):
    """SURVEY Appendix A SG KAT (compress_supergroup, w=4, chunk 2, slot 1 of 4, sg 5)."""
    v = np.array([(k - 128) / 64 + (k % 7) * 0.001 for k in range(256)], np.float32)
    q = dq.QuantContext(dq.SharedSeed(1, 0), chunk_index=2, hop_slot=1, n_slots=4)
    b = dq.serialize_chunk(dq.compress_chunk(torch.from_numpy(v).cuda(), [4], dq.CodecConfig(), q, 5))
    rec = b[24:]
    assert rec[0] | rec[1] << 8 == 0x4000
    assert list(rec[2:18]) == [255, 223, 191, 159, 128, 95, 63, 32, 30, 63, 93, 125, 158, 190, 222, 254]
    assert rec[18:34].hex() == "fffffdffdfffddddffffffdffddfffdd"


def test_zero_and_top_index(dq):
    """proj/tests/test_codec.cpp:44-67: zero SG encodes to zeros; entries == group max take the top index."""
    cfg = dq.CodecConfig()
    z = dq.compress_chunk(torch.zeros(256, device="cuda"), [4], cfg, dq.QuantContext(dq.SharedSeed(1)))
    assert int(z.data.sum()) == 0
    for w in (2, 4, 8):
        c = dq.compress_chunk(torch.full((256,), 2.5, device="cuda"), [w], cfg, dq.QuantContext(dq.SharedSeed(2)))
        rec = dq.serialize_chunk(c)[24 + 18:]
        top = (1 << (w - 1)) - 1
        bits = np.unpackbits(np.frombuffer(rec, np.uint8), bitorder="little").reshape(256, w)
        codes = (bits * (1 << np.arange(w))).sum(1)
        assert np.all(codes == top << 1)


def test_errors(dq):
    cfg = dq.CodecConfig()
    x = torch.zeros(512, device="cuda")
    with pytest.raises(dq.InvalidArgument):
        dq.compress_chunk(x, [4, 8], cfg, dq.QuantContext())  # unsorted body
    with pytest.raises(dq.InvalidArgument):
        dq.compress_chunk(x, [3, 3], cfg, dq.QuantContext())  # check_width (codec.cpp:15-18)
    with pytest.raises(dq.InvalidArgument):
        dq.compress_chunk(x, [16, 2], cfg, dq.QuantContext())  # passthrough run must be last
    with pytest.raises(dq.InvalidArgument):
        dq.compress_chunk(x, [4], cfg, dq.QuantContext())  # length mismatch
    with pytest.raises(dq.InvalidArgument):
        dq.compress_chunk(x[:256], [4], cfg, dq.QuantContext(hop_slot=3, n_slots=2))
