"""Device-side reference wire format (dq_serialize_chunk / dq_parse_chunk) against the
oracle's serialize_chunk bytes and the host strict parser (proj/src/codec.cpp:319-399;
proj/tests/test_codec.cpp:142-155 sizes, :209-222 bit flips)."""
import numpy as np
import pytest

from tests.golden.make_golden import det_values

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_08923_b200 as dq
    return dq


def _vals(seed, n):
    return det_values(seed, n) if n else np.zeros(0, np.float32)


def _widths(runs):
    runs = tuple(runs) + (0,) * (4 - len(runs))
    return [8] * runs[0] + [4] * runs[1] + [2] * runs[2] + [16] * runs[3]


def _ref_bytes(port, runs, seed=1):
    w = np.array(_widths(runs), np.uint8)
    v = _vals(seed, w.size * 256)
    return port.compress_chunk(v, w, port.codec(), port.qctx(seed, 0, 3, 1, 4, True), first_sg=2)


def _dev(b: bytes):
    return torch.tensor(np.frombuffer(b, np.uint8).copy(), dtype=torch.uint8, device="cuda")


RUNS = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (3, 5, 9), (65, 2, 64), (0, 130, 1), (200, 300, 500),
        (0, 0, 0, 1), (1, 2, 3, 4), (64, 0, 0, 65)]


@pytest.mark.parametrize("runs", RUNS)
def test_device_serialize_matches_oracle(dq, port, runs):
    """GPU compress -> GPU serialize == the oracle's compress_chunk wire bytes."""
    w = _widths(runs)
    v = _vals(1, len(w) * 256)
    ch = dq.compress_chunk(torch.from_numpy(v).cuda(), w, dq.CodecConfig(),
                           dq.QuantContext(dq.SharedSeed(1, 0), 3, 1, 4, True), first_sg_index=2)
    wire = dq.serialize_chunk(ch, device=True)
    assert bytes(wire.cpu().numpy()) == _ref_bytes(port, runs)
    assert bytes(wire.cpu().numpy()) == dq.serialize_chunk(ch)


@pytest.mark.parametrize("runs", RUNS)
def test_device_parse_matches_host(dq, port, runs):
    ref = _ref_bytes(port, runs)
    ci, n8, n4, n2, n16, soa = dq.soa_from_reference(ref)
    ch = dq.parse_chunk(_dev(ref))
    assert (ch.chunk_index, ch.n8, ch.n4, ch.n2, ch.n16) == (ci, n8, n4, n2, n16)
    assert np.array_equal(ch.data.cpu().numpy()[: soa.size], soa)
    assert bytes(dq.serialize_chunk(ch, device=True).cpu().numpy()) == ref


def _outcome(fn):
    import paper_2602_08923_b200 as dq
    try:
        r = fn()
        return ("ok", r)
    except (dq.MalformedBuffer, dq.InvalidArgument) as e:
        return (type(e).__name__, str(e))


def _same(dq, buf: bytes):
    host = _outcome(lambda: dq.soa_from_reference(buf))
    dev = _outcome(lambda: dq.parse_chunk(_dev(buf)))
    assert host[0] == dev[0], (host, dev)
    if host[0] == "ok":
        ci, n8, n4, n2, n16, soa = host[1]
        ch = dev[1]
        assert (ch.chunk_index, ch.n8, ch.n4, ch.n2, ch.n16) == (ci, n8, n4, n2, n16)
        assert np.array_equal(ch.data.cpu().numpy()[: soa.size], soa)
    else:
        assert host[1] == dev[1]
    return host[0]


def test_device_parse_malformed(dq, port):
    ref = _ref_bytes(port, (0, 1, 1), seed=9)
    for cut in (0, 1, 23, 24, 25, len(ref) // 2, len(ref) - 1):
        assert _same(dq, ref[:cut]) == "MalformedBuffer"
    assert _same(dq, ref + b"\0") == "MalformedBuffer"
    t = bytearray(ref)
    t[8] += 1  # run lengths no longer sum to the count
    assert _same(dq, bytes(t)) == "MalformedBuffer"
    t = bytearray(ref)
    t[20] = 1  # a width-16 run the body does not hold
    t[4] += 1
    assert _same(dq, bytes(t)) == "MalformedBuffer"
    p16 = _ref_bytes(port, (1, 0, 0, 2), seed=5)
    for cut in (len(p16) - 1, 24 + 100, 24 + 274 + 511):
        assert _same(dq, p16[:cut]) == "MalformedBuffer"
    zeros = port.compress_chunk(np.zeros(3 * 256, np.float32), np.array([8, 4, 2], np.uint8), port.codec(),
                                port.qctx(9))
    for pos, kind in ((24 + 2, "group scale"), (-1, "payload"), (24 + 274 + 146 + 5, "group scale")):
        z = bytearray(zeros)
        z[pos] = 0x10
        assert _same(dq, bytes(z)) == "MalformedBuffer"
        with pytest.raises(dq.MalformedBuffer, match=kind):
            dq.parse_chunk(_dev(bytes(z)))
    # first offending super-group decides, also when the buffer is truncated later
    z = bytearray(zeros)
    z[-1] = 1
    z[24 + 274 + 3] = 1
    assert _same(dq, bytes(z[:-5])) == "MalformedBuffer"
    with pytest.raises(dq.MalformedBuffer, match="group scale"):
        dq.parse_chunk(_dev(bytes(z[:-5])))


def test_device_parse_random_flips(dq, port):
    """test_codec.cpp:209-222: a flipped bit is rejected or re-serializes identically,
    with the same verdict and message as the host parser."""
    ref = _ref_bytes(port, (2, 2, 2, 2), seed=4)
    zeros = port.compress_chunk(np.zeros(6 * 256, np.float32), np.array([8, 8, 4, 4, 2, 2], np.uint8),
                                port.codec(), port.qctx(4))
    rng = np.random.default_rng(0)
    seen = set()
    for base in (ref, zeros):
        for _ in range(150):
            t = bytearray(base)
            pos = int(rng.integers(0, len(t)))
            t[pos] ^= 1 << int(rng.integers(0, 8))
            verdict = _same(dq, bytes(t))
            seen.add(verdict)
            if verdict == "ok":
                ch = dq.parse_chunk(_dev(bytes(t)))
                assert bytes(dq.serialize_chunk(ch, device=True).cpu().numpy()) == bytes(t)
    assert {"ok", "MalformedBuffer"} <= seen


def test_device_wire_roundtrip_large(dq):
    """Serialize -> parse -> serialize of a 2^16-super-group chunk is the identity."""
    g = torch.Generator(device="cuda").manual_seed(3)
    n8, n4, n2 = 9000, 20000, 36536
    x = torch.randn((n8 + n4 + n2) * 256, device="cuda", generator=g)
    w = np.repeat(np.array([8, 4, 2], np.uint8), [n8, n4, n2])
    ch = dq.compress_chunk(x, w, dq.CodecConfig(), dq.QuantContext(dq.SharedSeed(1, 0), 1, 0, 4, True))
    wire = dq.serialize_chunk(ch, device=True)
    assert wire.numel() == dq.wire_bytes(n8, n4, n2)
    back = dq.parse_chunk(wire)
    assert torch.equal(back.data[: ch.data.numel()], ch.data)
    assert torch.equal(dq.serialize_chunk(back, device=True), wire)
