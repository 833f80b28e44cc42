"""Parity at the BASELINE configs themselves (SURVEY §8 config notation).

* C1 — ring, n = 4, d = 2^24, b = 4, the reference's locality generator (σ_log = 4,
  generator seed 1, round seed {1, 0}; proj/src/synth.cpp:31-54): the device round's
  wire_hash (FNV over every transmitted byte, proj/src/engine.cpp:16-22,371-388) equals the
  SURVEY Appendix-A pin 55fe6ac1285215b7, and the synced gradient, widths, permutation,
  u and wire accounting equal the reference library's run_round bit for bit.
* C2 — the bench config (n = 4, d = 2^26): the same comparison against the reference's
  run_round (threads = 4).
* C3 — one chunk of the 8-GPU ring at 2^28 entries per rank, checked chunk-wise
  (SURVEY H8): every hop of chunk 3 (leaf, six fused DAR hops, the sink DAR) is compared
  byte for byte with the reference's compress_chunk / decompress_accumulate_recompress
  (proj/src/codec.cpp:164-183,238-266) under the same QuantContext, each hop fed the
  device's previous message (induction over the hops), with the statistics and the fast
  allocation of the full 2^20-super-group gradient compared with the reference first.

The oracle is the reference library compiled from its own sources (oracle/_ref) when
present, else the C restatement; both are checkers only.
"""
import concurrent.futures as cf

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

C1_WIRE_HASH = 0x55FE6AC1285215B7


@pytest.fixture(scope="module")
def dq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_08923_b200 as dq
    return dq


@pytest.fixture(scope="module")
def oracle():
    from oracle.oracle import Oracle, available
    return Oracle("reference" if available("reference") else "port")


def _generate(ora, n, d, seed=1, sigma_log=4.0):
    """proj/src/synth.cpp:31-54 for ranks 0..n-1, one thread per rank (ctypes drops the GIL)."""
    with cf.ThreadPoolExecutor(n) as ex:
        return list(ex.map(lambda r: ora.generate_worker(d, seed=seed, sigma_log=sigma_log, rank=r), range(n)))


def _round_vs_reference(dq, ora, n, d, pin=None):
    ws = _generate(ora, n, d)
    cfg = dq.PipelineConfig(n_workers=n, budget_bits=4.0, topology=dq.RING, seed=dq.SharedSeed(1, 0))
    got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg, collect_wire=True, with_allocation=True)
    synced = got.synced.cpu().numpy()
    if pin is not None:
        assert got.wire_hash == pin, hex(got.wire_hash)
    want = ora.run_round(ws, ora.round_cfg(n, 4.0, "ring", seed=1, threads=n))
    assert got.wire_hash == want["wire_hash"]
    assert np.array_equal(synced.view(np.uint32), want["synced"].view(np.uint32))
    assert np.array_equal(got.widths, want["widths"])
    assert np.array_equal(got.permutation, want["perm"])
    assert got.u == want["u"]
    assert got.payload_bits == want["payload_bits"]
    for k in ("stats_bits", "wire_payload_bits", "scale_bits", "header_bits", "repr_bits",
              "compressed_coordinates", "transmitted_coordinates"):
        assert got.info[k] == want[k], k
    # vNMSE: fp64 sums in a different order than the reference's sequential loop
    # (engine.cpp:409-416), so equal to ~1e-12 relative, not bit for bit
    assert got.vnmse == pytest.approx(want["vnmse"], rel=1e-10)
    return got, want


def test_c1_reference_config(dq, oracle):
    """C1: 4 x 2^24, ring, b = 4 -> wire_hash 55fe6ac1285215b7, u = -8.300096..., vNMSE 1.0584e-4."""
    got, want = _round_vs_reference(dq, oracle, 4, 1 << 24, pin=C1_WIRE_HASH)
    assert got.u == pytest.approx(-8.300096, abs=5e-7)
    assert got.vnmse == pytest.approx(1.058403e-4, rel=1e-6)
    assert got.u == want["u"]


@pytest.mark.slow
def test_c2_bench_config(dq, oracle):
    """C2 (the N = 1 bench config): 4 x 2^26, ring, b = 4, bit-exact vs the reference's run_round."""
    _round_vs_reference(dq, oracle, 4, 1 << 26)


def _locality_gpu(n, d, seed):
    """A σ_log = 4 locality gradient made on the GPU (shared per-super-group scale, per-rank
    entries); the oracle sees the same bytes, so any generator serves parity."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = d // 256
    scale = torch.exp(4.0 * torch.randn(T, 1, device="cuda", generator=g))
    return [(torch.randn(T, 256, device="cuda", generator=g) * scale).view(-1) for _ in range(n)]


@pytest.mark.slow
def test_c3_chunkwise_ring8(dq, oracle):
    """C3 chunk-wise: n = 8 ranks x 2^28 entries, ring, b = 4; chunk 3's eight compressions."""
    n, d, c = 8, 1 << 28, 3
    T = d // 256
    xs = _locality_gpu(n, d, seed=3)
    means, sqs = zip(*[dq.compute_stats(x) for x in xs])
    means, sqs = torch.stack(means), torch.stack(sqs)
    gm, gs = dq.reduce_stats(means, sqs)
    # statistics of one rank and the rank-ordered reduction vs the reference (stats.cpp:23-54)
    m0, q0 = oracle.compute_stats(xs[5].cpu().numpy())
    assert np.array_equal(means[5].cpu().numpy().view(np.uint32), m0.view(np.uint32))
    assert np.array_equal(sqs[5].cpu().numpy().view(np.uint32), q0.view(np.uint32))
    hm, hq = oracle.reduce_stats(means.cpu().numpy(), sqs.cpu().numpy())
    assert np.array_equal(gm.cpu().numpy().view(np.uint32), hm.view(np.uint32))
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), hq.view(np.uint32))
    # fast allocation over all 2^20 super-groups (allocation.cpp:228-260, 302-310)
    al = dq.allocate_fast(gs, 4.0)
    w_ref, p_ref, u_ref, pay_ref = oracle.allocate_fast(hq, 4.0)
    perm = al.permutation.cpu().numpy().astype(np.uint32)
    assert np.array_equal(al.widths.cpu().numpy(), w_ref)
    assert np.array_equal(perm, p_ref)
    assert al.u == u_ref and al.payload_bits == pay_ref
    # chunk c: permuted super-groups [T c / n, T (c+1) / n) (engine.cpp:52-62), normalized
    lo, hi = T * c // n, T * (c + 1) // n
    idx = al.permutation[lo:hi].long()
    w_chunk = w_ref[p_ref[lo:hi]]
    locals_ = [(x.view(T, 256)[idx] - gm[idx][:, None]).contiguous().view(-1) for x in xs]
    cfg = dq.CodecConfig()
    cc = oracle.codec(16, 256, True, True)

    def q(slot):
        return dq.QuantContext(dq.SharedSeed(1, 0), chunk_index=c, hop_slot=slot, n_slots=n)

    # ring schedule of chunk c (topology.cpp:8-27): hop h is sent by rank (c + 1 + h) % n at
    # slot h; the sink (rank c) recompresses at slot n - 1
    senders = [(c + 1 + h) % n for h in range(n - 1)] + [c]
    msgs = [dq.compress_chunk(locals_[senders[0]], w_chunk, cfg, q(0), lo)]
    for h in range(1, n):
        msgs.append(dq.decompress_accumulate_recompress(msgs[-1], locals_[senders[h]], cfg, q(h), lo))
    dev = [dq.serialize_chunk(m) for m in msgs]
    host_locals = [locals_[s].cpu().numpy() for s in senders]
    del locals_, xs

    def check(h):
        qc = oracle.qctx(1, 0, c, h, n, True)
        if h == 0:
            want = oracle.compress_chunk(host_locals[0], w_chunk, cc, qc, first_sg=lo)
        else:
            want = oracle.dar_chunk(dev[h - 1], host_locals[h], cc, qc, first_sg=lo)
        return h, want == dev[h]

    with cf.ThreadPoolExecutor(n) as ex:
        res = dict(ex.map(check, range(n)))
    assert all(res.values()), res
