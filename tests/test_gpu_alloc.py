"""Parity of the statistics and fast-allocation kernels with the oracle.

Cases follow proj/tests/test_stats.cpp and test_allocation.cpp: sequential fp64
stats, rank-ordered reduction, allocation boundary ties, no positive norms,
every flip within budget, infeasible budgets.
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


@pytest.mark.parametrize("d", [256, 1000, 1 << 16, (1 << 16) + 3])
def test_stats_match(dq, port, d):
    rng = np.random.default_rng(d)
    x = (rng.standard_normal(d) * np.exp(3 * rng.standard_normal(d))).astype(np.float32)
    m, q = dq.compute_stats(torch.from_numpy(x).cuda())
    mo, qo = port.compute_stats(x)
    assert np.array_equal(m.cpu().numpy().view(np.uint32), mo.view(np.uint32))
    assert np.array_equal(q.cpu().numpy().view(np.uint32), qo.view(np.uint32))


def test_reduce_stats_match(dq, port):
    rng = np.random.default_rng(1)
    means = rng.standard_normal((5, 3000)).astype(np.float32)
    sqs = np.abs(rng.standard_normal((5, 3000)) * 1e3).astype(np.float32)
    gm, gs = dq.reduce_stats(torch.from_numpy(means).cuda(), torch.from_numpy(sqs).cuda())
    om, os_ = port.reduce_stats(means, sqs)
    assert np.array_equal(gm.cpu().numpy().view(np.uint32), om.view(np.uint32))
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), os_.view(np.uint32))


def _F_cases():
    rng = np.random.default_rng(7)
    yield "lognormal", np.exp(8 * rng.standard_normal(50000)).astype(np.float32)
    yield "normal_sq", (rng.standard_normal(20000) ** 2 * 256).astype(np.float32)
    f = np.exp(4 * rng.standard_normal(10000)).astype(np.float32)
    f[::7] = 0.0
    yield "with_zeros", f
    yield "all_zero", np.zeros(1000, np.float32)
    yield "constant", np.full(4096, 3.0, np.float32)
    yield "two_levels", np.repeat(np.array([1.0, 1000.0], np.float32), 3000)
    yield "single", np.array([5.0], np.float32)
    yield "tiny", np.array([1e-30, 2e-30, 1e-20], np.float32)
    yield "ratio_ties", np.array([17.0, 512.0, 17.0 * 512 / 17, 1.0, 512 / 17], np.float32)
    g = np.exp(2 * rng.standard_normal(3000)).astype(np.float32)
    yield "dupes", np.concatenate([g, g, g])


@pytest.mark.parametrize("b", [2.6, 3, 4, 5, 6, 8, 12])
@pytest.mark.parametrize("name,F", list(_F_cases()), ids=[c[0] for c in _F_cases()])
def test_allocate_fast_matches(dq, port, name, F, b):
    from oracle.oracle import OracleError
    try:
        w, p, u, pay = port.allocate_fast(F, b)
    except OracleError as e:
        assert e.code == 3
        with pytest.raises(dq.InfeasibleBudget):
            dq.allocate_fast(torch.from_numpy(F).cuda(), b)
        return
    got = dq.allocate_fast(torch.from_numpy(F).cuda(), b)
    assert np.array_equal(got.widths.cpu().numpy(), w)
    assert np.array_equal(got.permutation.cpu().numpy().astype(np.uint32), p)
    assert got.u == u
    assert got.payload_bits == pay


def test_allocate_infeasible(dq):
    with pytest.raises(dq.InfeasibleBudget):
        dq.allocate_fast(torch.ones(100, device="cuda"), 2.0)


@pytest.mark.parametrize("seed", [5, 0])
def test_allocate_fast_float_threshold_near_tie(dq, port, seed):
    """At T = 2^22 a flip can sit within float rounding of the plateau's threshold, so the
    exact-arithmetic crossing and the reference's float-threshold bisection disagree
    (seed 5, found by tools/find_alloc_ties.py; seed 0 agrees).  The device must still
    return the reference's allocation."""
    rng = np.random.default_rng(seed)
    F = (np.exp(8 * rng.standard_normal(1 << 22)) * 256).astype(np.float32)
    w, p, u, pay = port.allocate_fast(F, 4.0)
    got = dq.allocate_fast(torch.from_numpy(F).cuda(), 4.0)
    assert got.u == u
    assert got.payload_bits == pay
    assert np.array_equal(got.widths.cpu().numpy(), w)
    assert np.array_equal(got.permutation.cpu().numpy().astype(np.uint32), p)


@pytest.mark.parametrize("b", [2.6, 3, 4, 6, 12])
@pytest.mark.parametrize("name,F", list(_F_cases()), ids=[c[0] for c in _F_cases()])
def test_allocate_general_matches(dq, port, name, F, b):
    """allocate_general (allocation.cpp:121-168), W = {2,4,8}: widths, permutation,
    resolved base threshold and payload identical to the oracle."""
    from oracle.oracle import OracleError
    try:
        w, p, u, pay = port.allocate_general(F, b)
    except OracleError as e:
        assert e.code == 3
        with pytest.raises(dq.InfeasibleBudget):
            dq.allocate_general(torch.from_numpy(F).cuda(), b)
        return
    got = dq.allocate_general(torch.from_numpy(F).cuda(), b)
    assert np.array_equal(got.widths.cpu().numpy(), w)
    assert np.array_equal(got.permutation.cpu().numpy().astype(np.uint32), p)
    assert got.u == u
    assert got.payload_bits == pay


def test_allocate_general_large_and_collisions(dq, port):
    rng = np.random.default_rng(9)
    f = (np.exp(5 * rng.standard_normal(1 << 18)) * 64).astype(np.float32)
    F = np.concatenate([f, (f.astype(np.float64) * (512 / 17)).astype(np.float32), f[:1000]])
    for b in (3.3, 4, 5.5):
        w, p, u, pay = port.allocate_general(F, b)
        got = dq.allocate_general(torch.from_numpy(F).cuda(), b)
        assert got.u == u and got.payload_bits == pay
        assert np.array_equal(got.widths.cpu().numpy(), w)
        assert np.array_equal(got.permutation.cpu().numpy().astype(np.uint32), p)


def test_allocate_general_rejects_negative(dq):
    for bad in (np.array([1.0, -1.0], np.float32), np.array([np.nan, 1.0], np.float32)):
        with pytest.raises(dq.InvalidArgument):
            dq.allocate_general(torch.from_numpy(bad).cuda(), 5.0)


def test_allocate_fast_stateful_sequence(dq, port):
    """allocate_fast_stateful (allocation.cpp:262-300) over 12 rounds with the state carried:
    widths, permutation, reported u, payload and the next state identical to the oracle."""
    rng = np.random.default_rng(5)
    for b in (3, 4, 6):
        st = dq.FastAllocatorState()
        ost = [-1e6, 1e6, 0.0]
        for rnd in range(12):
            F = np.exp((4 + rnd % 3) * rng.standard_normal(1500)).astype(np.float32)
            w, p, u, pay, ost = port.allocate_fast_stateful(F, b, ost)
            got = dq.allocate_fast_stateful(torch.from_numpy(F).cuda(), b, st)
            assert np.array_equal(got.widths.cpu().numpy(), w)
            assert np.array_equal(got.permutation.cpu().numpy().astype(np.uint32), p)
            assert got.u == u and got.payload_bits == pay
            assert [st.lo, st.hi, st.u] == ost
