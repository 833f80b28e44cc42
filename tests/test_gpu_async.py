"""Asynchronous rounds: the fast allocation decided and certified on the device, no host
synchronisation inside a round.

* bit-identical to the oracle's run_round (proj/src/engine.cpp:269-418): synced gradient,
  widths, permutation, u, payload and wire accounting - without the wire-hash mode, which
  forces the host-synchronous path;
* the rare rounds the device cannot certify, forced: the context's host service thread
  finishes the allocation from the exported F (allocation.cpp:195-260) and releases the
  assignment;
* metrics=False returns at once; Context.wait() fills the allocation fields later;
* a whole round captured in a CUDA graph and replayed on new inputs equals direct rounds.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_08923_b200 as dq
    return dq


def _workers(port, n, d, seed, sigma_log=4.0):
    return [port.generate_worker(d, seed=seed, sigma_log=sigma_log, rank=r) for r in range(n)]


def _cfg(dq, n, b, topo="ring", seed=1):
    return dq.PipelineConfig(n_workers=n, budget_bits=b, topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING,
                             seed=dq.SharedSeed(seed, 0))


def _check(dq, got, want):
    synced = got.synced.cpu().numpy()
    assert np.array_equal(synced.view(np.uint32), want["synced"].view(np.uint32))
    assert np.array_equal(got.widths, want["widths"])
    assert np.array_equal(got.permutation, want["perm"])
    assert got.u == want["u"]
    assert got.payload_bits == want["payload_bits"]
    for k in ("stats_bits", "wire_payload_bits", "scale_bits", "header_bits", "repr_bits",
              "compressed_coordinates", "transmitted_coordinates"):
        assert got.info[k] == want[k], k


@pytest.mark.parametrize("n,b,topo,d", [(4, 4.0, "ring", 1 << 16), (8, 3.0, "butterfly", (1 << 15) + 77),
                                        (3, 5.0, "ring", 1 << 14), (2, 6.0, "ring", 3000),
                                        # T = 4096 (largest one-CTA allocation) and 4097 (cooperative search)
                                        (4, 4.0, "ring", 1 << 20), (2, 3.0, "ring", (1 << 20) + 256),
                                        (4, 4.0, "ring", 1 << 22)])
def test_async_round_matches_oracle(dq, port, n, b, topo, d):
    ws = _workers(port, n, d, seed=11 + n)
    want = port.run_round(ws, port.round_cfg(n, b, topo, seed=1))
    got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], _cfg(dq, n, b, topo), with_allocation=True)
    _check(dq, got, want)


@pytest.mark.parametrize("n,b,d", [(4, 4.0, 1 << 16), (4, 5.0, (1 << 14) + 9), (8, 4.0, 1 << 15),
                                    (4, 4.0, (1 << 20) + 256)])
def test_host_finished_allocation(dq, port, n, b, d):
    """need_host forced on every round: the host service thread answers, the assignment
    waits for it; results unchanged (T <= 4096: the one-CTA allocation; larger: the
    cooperative search)."""
    from paper_2602_08923_b200._lib import check, lib
    ws = _workers(port, n, d, seed=23 + n)
    want = port.run_round(ws, port.round_cfg(n, b, "ring", seed=1))
    check(lib().dq_debug_force_host_alloc(1))
    try:
        got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], _cfg(dq, n, b), with_allocation=True)
    finally:
        check(lib().dq_debug_force_host_alloc(0))
    _check(dq, got, want)


def test_no_metrics_round_then_wait(dq, port):
    n, d = 4, 1 << 15
    ws = _workers(port, n, d, seed=5)
    want = port.run_round(ws, port.round_cfg(n, 4.0, "ring", seed=1))
    cfg = _cfg(dq, n, 4.0)
    ctx = dq.Context(cfg)
    r = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg, ctx=ctx, metrics=False)
    info = ctx.wait()
    assert np.array_equal(r.synced.cpu().numpy().view(np.uint32), want["synced"].view(np.uint32))
    assert info["u"] == want["u"] and info["payload_bits"] == want["payload_bits"]
    assert info["repr_bits"] == want["repr_bits"]
    assert info["n8"] * 8 + info["n4"] * 4 + info["n2"] * 2 == want["payload_bits"] // 256
    ctx.close()


def test_round_captured_in_cuda_graph(dq, port):
    """A simulated round (stats -> device allocation -> hops -> decode) captured once and
    replayed on new inputs equals direct rounds on those inputs."""
    n, d = 4, 1 << 16
    cfg = _cfg(dq, n, 4.0)
    ctx = dq.Context(cfg)
    xs = [torch.empty(d, device="cuda") for _ in range(n)]
    out = torch.empty(d, device="cuda")
    first = _workers(port, n, d, seed=41)
    for x, w in zip(xs, first):
        x.copy_(torch.from_numpy(w))
    dq.run_round(xs, cfg, out=out, ctx=ctx, metrics=False)  # sizes every buffer
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dq.run_round(xs, cfg, out=out, ctx=ctx, metrics=False)
    for seed in (41, 42, 43):
        ws = _workers(port, n, d, seed=seed)
        for x, w in zip(xs, ws):
            x.copy_(torch.from_numpy(w))
        g.replay()
        torch.cuda.synchronize()
        want = port.run_round(ws, port.round_cfg(n, 4.0, "ring", seed=1))
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want["synced"].view(np.uint32)), seed
    del g
    ctx.close()


@pytest.mark.parametrize("n,b,d", [(4, 4.0, 1 << 21), (2, 3.0, (1 << 20) + 256), (8, 4.0, (1 << 20) + 4096 * 3)])
def test_threshold_consult(dq, port, n, b, d):
    """Forced threshold consult (the path of a float threshold within rounding of an F_j):
    the host service thread answers the candidates' glibc u and thresholds, the device
    recounts and decides - results unchanged, no host-finished allocation."""
    from paper_2602_08923_b200._lib import check, lib
    ws = _workers(port, n, d, seed=31 + n)
    want = port.run_round(ws, port.round_cfg(n, b, "ring", seed=1))
    cfg = _cfg(dq, n, b)
    ctx = dq.Context(cfg)
    check(lib().dq_debug_force_host_alloc(2))
    try:
        got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg, ctx=ctx, with_allocation=True)
    finally:
        check(lib().dq_debug_force_host_alloc(0))
    _check(dq, got, want)
    h = ctx.host_allocations()
    assert h["finished"] == 0 and h["consulted"] >= 1, h
    ctx.close()


@pytest.mark.parametrize("n,d", [(2, 1 << 26), (2, 1 << 28), (4, 1 << 26)])
def test_large_rounds_decided_on_device(dq, n, d):
    """Bench-sized heavy-tailed gradients (dense F: adjacent-float F_j around the plateau
    are common) - every asynchronous round decided on the device (at most a threshold
    consult), bit-identical to the host-synchronous allocation path."""
    import os
    import bench
    cfg = _cfg(dq, n, 4.0)
    xs = bench.synth(torch, d, n, 4.0, seed=7)
    ctx = dq.Context(cfg)
    os.environ["DQ_SYNC_ALLOC"] = "1"
    try:
        ref_ctx = dq.Context(cfg)
    finally:
        del os.environ["DQ_SYNC_ALLOC"]
    for rnd in range(3):
        cfg.seed = dq.SharedSeed(1, rnd)
        ctx.set_config(cfg)
        ref_ctx.set_config(cfg)
        a = dq.run_round(xs, cfg, ctx=ctx, metrics=False).synced
        info = ctx.wait()
        r = dq.run_round(xs, cfg, ctx=ref_ctx, with_allocation=True)
        assert torch.equal(a.view(torch.int32), r.synced.view(torch.int32)), rnd
        assert info["u"] == r.u and info["payload_bits"] == r.payload_bits
    h = ctx.host_allocations()
    assert h["finished"] == 0, h
    print("host consults", h)
    ctx.close()
    ref_ctx.close()
