"""Full-round parity: device run_round (all workers on one GPU) vs the oracle's run_round.

Bit-exact: synced gradient, wire_hash over every transmitted byte (reference
wire format), widths, permutation, fast-allocator u and payload, wire
accounting.  Inputs come from the reference's own generator (restated in the
oracle) so the cases read like proj/tests/test_engine.cpp.
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


def _workers(port, n, d, seed, sigma_log=4.0, kind="locality"):
    return [port.generate_worker(d, seed=seed, sigma_log=sigma_log, rank=r, kind=kind) for r in range(n)]


def _cfg(dq, n, b, topo, seed=1, **kw):
    return dq.PipelineConfig(n_workers=n, budget_bits=b, topology=dq.BUTTERFLY if topo == "butterfly" else dq.RING,
                             seed=dq.SharedSeed(seed, 0), **kw)


def _check_round(dq, port, ws, cfg, ocfg):
    want = port.run_round(ws, ocfg)
    got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg, collect_wire=True, with_allocation=True)
    synced = got.synced.cpu().numpy()
    assert np.array_equal(synced.view(np.uint32), want["synced"].view(np.uint32))
    assert got.wire_hash == want["wire_hash"]
    assert np.array_equal(got.widths, want["widths"])
    assert np.array_equal(got.permutation, want["perm"])
    assert got.u == want["u"]
    assert got.payload_bits == want["payload_bits"]
    for k in ("stats_bits", "wire_payload_bits", "scale_bits", "header_bits", "repr_bits",
              "compressed_coordinates", "transmitted_coordinates"):
        assert got.info[k] == want[k], k
    assert got.vnmse == pytest.approx(want["vnmse"], rel=1e-9, abs=1e-15)
    return got, want


@pytest.mark.parametrize("topo", ["ring", "butterfly"])
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("b", [3, 4, 6])
def test_round_matches_oracle(dq, port, topo, n, b):
    d = 1 << 15
    ws = _workers(port, n, d, seed=13 + n)
    _check_round(dq, port, ws, _cfg(dq, n, b, topo), port.round_cfg(n, b, topo, seed=1))


@pytest.mark.parametrize("n,topo", [(16, "ring"), (16, "butterfly"), (12, "ring")])
def test_more_than_eight_workers(dq, port, n, topo):
    """n_slots > 8 takes the runtime-n permutation path of the fused kernels."""
    d = 1 << 14
    ws = _workers(port, n, d, seed=31)
    _check_round(dq, port, ws, _cfg(dq, n, 4, topo, seed=6), port.round_cfg(n, 4, topo, seed=6))


@pytest.mark.parametrize("n", [3, 5, 7])
def test_ring_odd_worker_counts(dq, port, n):
    d = (1 << 14) + 77  # padding in the last super-group
    ws = _workers(port, n, d, seed=3)
    _check_round(dq, port, ws, _cfg(dq, n, 5, "ring", seed=4), port.round_cfg(n, 5, "ring", seed=4))


@pytest.mark.parametrize("sigma_log,kind", [(1.0, "locality"), (0.0, "iid")])
def test_round_generators(dq, port, sigma_log, kind):
    d = 1 << 15
    ws = _workers(port, 4, d, seed=9, sigma_log=sigma_log, kind=kind)
    _check_round(dq, port, ws, _cfg(dq, 4, 4, "ring"), port.round_cfg(4, 4, "ring"))


def test_round_ablation_toggles(dq, port):
    d = 1 << 14
    ws = _workers(port, 4, d, seed=21)
    for kw in [dict(correlated=False), dict(non_uniform=False),
               dict(variable_width=False, allocator=dq.KIND_FIXED, fixed_width=4),
               dict(variable_width=False, allocator=dq.KIND_FIXED, fixed_width=2, correlated=False)]:
        okw = {k: v for k, v in kw.items() if k != "allocator"}
        if "allocator" in kw:
            okw["allocator"] = "fixed"
        _check_round(dq, port, ws, _cfg(dq, 4, 6, "ring", **kw), port.round_cfg(4, 6, "ring", **okw))


@pytest.mark.parametrize("topo,n,b", [("ring", 4, 4), ("butterfly", 8, 3), ("ring", 5, 6)])
def test_round_general_allocator(dq, port, topo, n, b):
    """AllocatorKind::kGeneral in run_round (engine.cpp:322-323), W = {2,4,8}."""
    d = (1 << 15) + 3
    ws = _workers(port, n, d, seed=40 + n)
    _check_round(dq, port, ws, _cfg(dq, n, b, topo, seed=2, allocator=dq.KIND_GENERAL),
                 port.round_cfg(n, b, topo, seed=2, allocator="general"))


@pytest.mark.parametrize("topo", ["ring", "butterfly"])
@pytest.mark.parametrize("s,hier", [(16, False), (32, False), (8, True), (32, True), (64, False), (128, True)])
def test_round_scale_formats(dq, port, s, hier, topo):
    """CodecConfig ablations on the device: group size s and flat bf16 group scales
    (codec.cpp:88-116,146-149; wire records without sg_scale, engine accounting 16/s)."""
    d = (1 << 14) + 9
    ws = _workers(port, 4, d, seed=60 + s)
    _check_round(dq, port, ws, _cfg(dq, 4, 5, topo, seed=3, group_size=s, hierarchical_scales=hier),
                 port.round_cfg(4, 5, topo, seed=3, s=s, hierarchical=hier))


def test_ablation_ladder(dq, port):
    """proj/tests/test_engine.cpp:241-260 on the device: every rung of ablation_ladder
    (engine.cpp:420-450) bit-identical to the oracle, mean vNMSE strictly decreasing."""
    ladder = dq.ablation_ladder(dq.PipelineConfig(n_workers=4, seed=dq.SharedSeed(0, 0)))
    assert [name for name, _ in ladder] == ["uniform", "non_uniform", "variable_width", "hierarchical", "correlated"]
    means = [0.0] * 5
    for smp in range(3):
        ws = _workers(port, 4, 1 << 16, seed=50 + smp)
        for v, (name, cfg) in enumerate(ladder):
            from dataclasses import replace
            cfg = replace(cfg, seed=dq.SharedSeed(70 + smp, 0))
            ocfg = port.round_cfg(4, cfg.budget_bits, "ring", seed=70 + smp, s=cfg.group_size,
                                  non_uniform=cfg.non_uniform, variable_width=cfg.variable_width,
                                  hierarchical=cfg.hierarchical_scales, correlated=cfg.correlated,
                                  fixed_width=cfg.fixed_width,
                                  allocator={0: "general", 1: "fast", 2: "fixed"}[cfg.allocator])
            got, _ = _check_round(dq, port, ws, cfg, ocfg)
            means[v] += got.vnmse
    assert all(means[v] < means[v - 1] for v in range(1, 5)), means


def test_round_known_answer_c1(dq, port):
    """SURVEY Appendix A round pins at d = 2^20 (n=4 ring b=4, b=5; n=8 ring/butterfly b=4)."""
    d = 1 << 20
    ws8 = _workers(port, 8, d, seed=1)
    pins = [(4, 4, "ring", 0x4a094af6775201da), (4, 5, "ring", 0xae9e4b918ba61cfa),
            (8, 4, "ring", 0xbeab00622d7ed622), (8, 4, "butterfly", 0xc9cd215e5cad079e)]
    for n, b, topo, h in pins:
        got = dq.run_round([torch.from_numpy(w).cuda() for w in ws8[:n]], _cfg(dq, n, b, topo), collect_wire=True)
        assert got.wire_hash == h, (n, b, topo, hex(got.wire_hash))


def test_single_worker_is_noop(dq, port):
    ws = _workers(port, 1, 4096, seed=5)
    got = dq.run_round([torch.from_numpy(ws[0]).cuda()], _cfg(dq, 1, 5, "ring"))
    assert np.array_equal(got.synced.cpu().numpy(), ws[0])
    assert got.vnmse == 0.0


def test_infeasible_budget(dq, port):
    ws = _workers(port, 2, 4096, seed=5)
    with pytest.raises(dq.InfeasibleBudget):
        dq.run_round([torch.from_numpy(w).cuda() for w in ws], _cfg(dq, 2, 2, "ring"))


def test_full_size_properties(dq):
    """64M entries x 4 workers (BASELINE config 2): deterministic, unbiased-ish, budget respected."""
    g = torch.Generator(device="cuda").manual_seed(0)
    d = 1 << 26
    scale = torch.exp(4.0 * torch.randn(d // 256, device="cuda", generator=g)).repeat_interleave(256)
    ws = [torch.randn(d, device="cuda", generator=g) * scale for _ in range(4)]
    cfg = _cfg(dq, 4, 4, "ring")
    a = dq.run_round(ws, cfg)
    a_sync = a.synced.clone()
    b = dq.run_round(ws, cfg)
    assert torch.equal(a_sync, b.synced)
    assert a.vnmse < 1e-3
    assert a.payload_bits <= d * (4 - 0.5625)
    assert torch.isfinite(a_sync).all()


def test_every_device_of_one_process(dq, port):
    """Codebooks and codec tables exist once per device: a context on device 1 created
    after device 0 was used in the same process must compute the same round."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs in one process")
    d = 1 << 14
    ws = _workers(port, 4, d, seed=77)
    want = port.run_round(ws, port.round_cfg(4, 4, "ring", seed=1))
    for dev in (0, 1):
        cfg = _cfg(dq, 4, 4, "ring")
        ctx = dq.Context(cfg, device=dev)
        with torch.cuda.device(dev):
            got = dq.run_round([torch.from_numpy(w).cuda(dev) for w in ws], cfg, collect_wire=True, ctx=ctx)
            synced = got.synced.cpu().numpy()
        assert np.array_equal(synced.view(np.uint32), want["synced"].view(np.uint32)), dev
        assert got.wire_hash == want["wire_hash"], dev
        ctx.close()
