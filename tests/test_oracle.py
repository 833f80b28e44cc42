"""Pins the CPU oracle (C restatement) before it is trusted as the checker.

1. Known-answer vectors from SURVEY.md Appendix A (measured on the reference).
2. Golden fixtures generated from the reference library (tests/golden/golden.json,
   made by tests/golden/make_golden.py from oracle/_ref).
3. Live comparison with the reference library when oracle/_ref is built.
4. The reference's own property tests (proj/tests/test_codec.cpp, test_random.cpp,
   test_allocation.cpp) re-run against the restatement.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.oracle import OracleError
from tests.golden.make_golden import det_values

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def f32sha(a) -> str:
    return sha(np.ascontiguousarray(a, np.float32).tobytes())


# ----------------------------------------------------------------- 1. KATs
def test_prng_known_answers(port):
    assert port.random_bits(1, 0, 1, 0, 0, 0) == 0x29ebe7305c62cc09
    assert port.random_bits(1, 0, 3, 2, 5, 7) == 0x7d68649d7a83df8d
    assert port.uniform_at(1, 0, 2, 0, 3, 1 | (2 << 32)) == 0.67447497154491809
    assert [port.permutation_slot(1, 0, 3, 0, 0, 0, s, 8) for s in range(8)] == [4, 0, 1, 3, 6, 7, 5, 2]
    want = [0.52046948067031573, 0.11022667922886671, 0.22025639133920422, 0.41077827099557118,
            0.86345458681984844, 0.96763499956606003, 0.74933338887331269, 0.33204452245689919]
    assert [port.correlated_uniform(1, 0, 1, 0, 0, 0, s, 8) for s in range(8)] == want


def test_codebook_known_answers(port):
    b4 = [float(x).hex() for x in port.codebook(4)]
    assert b4 == [float.fromhex(h).hex() for h in
                  ["0x0p+0", "0x1.8fc83ep-4", "0x1.a8c4c2p-3", "0x1.52e0bcp-2", "0x1.e12ee4p-2", "0x1.40a368p-1",
                   "0x1.9ab0dcp-1", "0x1p+0"]]
    assert list(port.codebook(2)) == [0.0, 1.0]
    b8 = port.codebook(8)
    assert [float(x).hex() for x in b8[:4]] == [float.fromhex(h).hex() for h in
                                                 ["0x0p+0", "0x1.72a998p-8", "0x1.7396dp-7", "0x1.1763ap-6"]]
    assert float(b8[-2]).hex() == float.fromhex("0x1.fa9244p-1").hex() and b8[-1] == 1.0


def test_sg_known_answer(port):
    v = np.array([(k - 128) / 64 + (k % 7) * 0.001 for k in range(256)], np.float32)
    b = port.compress_chunk(v, [4], port.codec(), port.qctx(1, 0, 2, 1, 4, True), first_sg=5)
    rec = b[24:]
    assert rec[0] | rec[1] << 8 == 0x4000
    assert list(rec[2:18]) == [255, 223, 191, 159, 128, 95, 63, 32, 30, 63, 93, 125, 158, 190, 222, 254]
    assert rec[18:34].hex() == "fffffdffdfffddddffffffdffddfffdd"


def test_payload_budget_known_answers(port):
    F = np.ones(64, np.float32)
    for b, ok in [(2, False), (3, True), (4, True), (5, True), (6, True)]:
        if ok:
            port.allocate_fast(F, b)
        else:
            with pytest.raises(OracleError) as e:
                port.allocate_fast(F, b)
            assert e.value.code == 3


# --------------------------------------------------------------- 2. golden
def test_golden_prng(port):
    for s, r, p, c, sg, e, want in GOLD["random_bits"]:
        assert port.random_bits(s, r, p, c, sg, e) == want
    for s, r, p, c, sg, e, want in GOLD["uniform_at"]:
        assert port.uniform_at(s, r, p, c, sg, e).hex() == want
    for n, want in GOLD["permutation"].items():
        assert [port.permutation_slot(1, 0, 3, 0, 0, 0, s, int(n)) for s in range(int(n))] == want
    assert [port.correlated_uniform(1, 0, 1, 0, 0, 0, s, 8).hex() for s in range(8)] == GOLD["correlated_uniform"]
    for key, want in GOLD["codebooks"].items():
        w, u = key.split("_")
        assert [float(x).hex() for x in port.codebook(int(w), u == "nu")] == want


@pytest.mark.parametrize("i", range(6))
def test_golden_codec(port, i):
    c = GOLD["codec"][i]
    runs = c["runs"]
    w = np.array([8] * runs[0] + [4] * runs[1] + [2] * runs[2], np.uint8)
    v = det_values(c["seed_values"], w.size * 256)
    loc = det_values(c["seed_local"], w.size * 256)
    cc = port.codec(16, 256, True, c["non_uniform"])
    q0 = port.qctx(c["seed"], c["round"], c["chunk"], c["slot"], c["n_slots"], c["correlated"])
    comp = port.compress_chunk(v, w, cc, q0, first_sg=c["first_sg"])
    assert sha(comp) == c["compress_sha"] and comp[:64].hex() == c["compress_head"]
    q1 = port.qctx(c["seed"], c["round"], c["chunk"], c["dar_slot"], c["n_slots"], c["correlated"])
    assert sha(port.dar_chunk(comp, loc, cc, q1, first_sg=c["first_sg"])) == c["dar_sha"]
    assert f32sha(port.decompress_chunk(comp, cc, v.size)) == c["decompress_sha"]
    assert f32sha(port.decompress_accumulate(comp, cc, loc)) == c["da_sha"]


def test_golden_stats(port):
    for s in GOLD["stats"]:
        m, q = port.compute_stats(det_values(s["seed"], s["d"]))
        assert f32sha(m) == s["mean_sha"] and f32sha(q) == s["sq_sha"]


def golden_F():
    rng = np.random.default_rng(GOLD["allocation_inputs"]["rng_seed"])
    return {"lognormal": np.exp(8 * rng.standard_normal(3000)).astype(np.float32),
            "zeros_mixed": np.where(rng.random(2000) < 0.2, 0, np.exp(3 * rng.standard_normal(2000))).astype(np.float32),
            "constant": np.full(500, 3.0, np.float32)}


def test_golden_allocation(port):
    Fs = golden_F()
    for a in GOLD["allocation"]:
        F = Fs[a["name"]]
        assert f32sha(F) == a["F_sha"]
        w, p, u, pay = port.allocate_fast(F, a["b"])
        assert sha(w.tobytes()) == a["widths_sha"] and sha(p.astype(np.uint32).tobytes()) == a["perm_sha"]
        assert u.hex() == a["u"] and pay == a["payload_bits"]


def test_golden_general_allocation(port):
    Fs = golden_F()
    for a in GOLD["allocation_general"]:
        w, p, u, pay = port.allocate_general(Fs[a["name"]], a["b"], tuple(a["W"]))
        assert sha(w.tobytes()) == a["widths_sha"] and sha(p.astype(np.uint32).tobytes()) == a["perm_sha"]
        assert u.hex() == a["u"] and pay == a["payload_bits"]


def test_golden_rounds(port):
    for g in GOLD["rounds"]:
        ws = [port.generate_worker(g["d"], seed=g["seed"], sigma_log=4.0, rank=r) for r in range(g["n"])]
        assert sha(b"".join(w.tobytes() for w in ws)) == g["inputs_sha"]
        res = port.run_round(ws, port.round_cfg(g["n"], g["b"], g["topology"], seed=g["seed"],
                                                allocator=g.get("allocator", "fast")))
        assert f"{res['wire_hash']:016x}" == g["wire_hash"]
        assert f32sha(res["synced"]) == g["synced_sha"]
        assert sha(res["widths"].tobytes()) == g["widths_sha"] and sha(res["perm"].tobytes()) == g["perm_sha"]
        assert res["u"].hex() == g["u"] and res["payload_bits"] == g["payload_bits"]
        assert res["vnmse"].hex() == g["vnmse"]


# ------------------------------------------------------ 3. live vs _ref
@pytest.mark.parametrize("trial", range(4))
def test_live_codec_vs_reference(port, ref, trial):
    rng = np.random.default_rng(1000 + trial)
    runs = tuple(int(x) for x in rng.integers(0, 6, 3))
    if sum(runs) == 0:
        runs = (1, 1, 1)
    w = np.array([8] * runs[0] + [4] * runs[1] + [2] * runs[2], np.uint8)
    v = det_values(5000 + trial, w.size * 256)
    loc = det_values(6000 + trial, w.size * 256)
    for nsl in (1, 2, 5, 8):
        for slot in {0, nsl - 1, nsl // 2}:
            for corr in (True, False):
                cc = port.codec()
                q = port.qctx(trial, 1, 2, slot, nsl, corr)
                a = port.compress_chunk(v, w, cc, q, first_sg=trial)
                assert a == ref.compress_chunk(v, w, cc, q, first_sg=trial)
                assert port.dar_chunk(a, loc, cc, q, first_sg=trial) == ref.dar_chunk(a, loc, cc, q, first_sg=trial)


@pytest.mark.parametrize("topo,n,b", [("ring", 4, 4), ("ring", 5, 3), ("butterfly", 4, 6), ("butterfly", 8, 4)])
def test_live_round_vs_reference(port, ref, topo, n, b):
    d = 3 * (1 << 12) + 5
    ws = [ref.generate_worker(d, seed=n, sigma_log=1.0, rank=r) for r in range(n)]
    for kw in [{}, {"correlated": False}, {"non_uniform": False}]:
        cfg = port.round_cfg(n, b, topo, seed=2, **kw)
        x, y = port.run_round(ws, cfg), ref.run_round(ws, cfg)
        for k in x:
            if isinstance(x[k], np.ndarray):
                assert np.array_equal(x[k], y[k]), k
            else:
                assert x[k] == y[k], k


def test_live_allocation_vs_reference(port, ref):
    rng = np.random.default_rng(3)
    for F in [np.exp(6 * rng.standard_normal(5000)).astype(np.float32), np.zeros(10, np.float32),
              np.array([1e-30, 5e-31], np.float32), np.repeat(np.float32(7.0), 33)]:
        for b in (2.7, 3, 4.5, 8):
            try:
                want = ref.allocate_fast(F, b)
            except OracleError as e:
                with pytest.raises(OracleError) as e2:
                    port.allocate_fast(F, b)
                assert e2.value.code == e.code
                continue
            got = port.allocate_fast(F, b)
            for a, c in zip(got, want):
                assert np.array_equal(a, c)


def _general_cases():
    rng = np.random.default_rng(11)
    yield np.exp(6 * rng.standard_normal(3000)).astype(np.float32)
    yield np.zeros(10, np.float32)
    yield np.array([1e-30, 5e-31, 0.0], np.float32)
    yield np.repeat(np.float32(7.0), 33)
    f = np.exp(3 * rng.standard_normal(2000)).astype(np.float32)
    yield np.concatenate([f, f * np.float32(512 / 17), f])  # points colliding across the chain


@pytest.mark.parametrize("W", [(2, 4, 8), (1, 2, 4, 8, 16), (4,), (2, 8), (1, 2), (2, 4, 8, 16)])
def test_live_general_allocation_vs_reference(port, ref, W):
    """proj/src/allocation.cpp:121-168 (allocate_general), every width set it accepts."""
    for F in _general_cases():
        for b in (2.2, 3, 4.5, 8, 17):
            for hier in (True, False):
                try:
                    want = ref.allocate_general(F, b, W, hierarchical=hier)
                except OracleError as e:
                    with pytest.raises(OracleError) as e2:
                        port.allocate_general(F, b, W, hierarchical=hier)
                    assert e2.value.code == e.code
                    continue
                got = port.allocate_general(F, b, W, hierarchical=hier)
                for a, c in zip(got, want):
                    assert np.array_equal(a, c)


def test_general_allocation_rejects_like_reference(port, ref):
    F = np.ones(8, np.float32)
    for W, Fx in [((2, 4, 3), F), ((3,), F), ((), F), ((2, 4, 8), np.array([1, -1], np.float32)),
                  ((2, 4, 8), np.array([np.nan], np.float32))]:
        with pytest.raises(OracleError) as a:
            ref.allocate_general(Fx, 5, W)
        with pytest.raises(OracleError) as c:
            port.allocate_general(Fx, 5, W)
        assert a.value.code == c.value.code == 2


def test_live_stateful_fast_vs_reference(port, ref):
    """proj/src/allocation.cpp:262-300: the carried u, its projection and the bisection step."""
    rng = np.random.default_rng(5)
    for b in (3, 4, 6):
        s_port = s_ref = [-1e6, 1e6, 0.0]
        for rnd in range(12):
            F = np.exp((4 + rnd % 3) * rng.standard_normal(1500)).astype(np.float32)
            try:
                want = ref.allocate_fast_stateful(F, b, s_ref)
            except OracleError as e:
                with pytest.raises(OracleError) as e2:
                    port.allocate_fast_stateful(F, b, s_port)
                assert e2.value.code == e.code
                continue
            got = port.allocate_fast_stateful(F, b, s_port)
            for a, c in zip(got[:4], want[:4]):
                assert np.array_equal(a, c)
            assert got[4] == want[4]
            s_port, s_ref = got[4], want[4]


@pytest.mark.parametrize("topo,n,b", [("ring", 4, 4), ("butterfly", 4, 3)])
def test_live_round_general_allocator_vs_reference(port, ref, topo, n, b):
    d = 3 * (1 << 12) + 5
    ws = [ref.generate_worker(d, seed=n, sigma_log=2.0, rank=r) for r in range(n)]
    cfg = port.round_cfg(n, b, topo, seed=2, allocator="general")
    x, y = port.run_round(ws, cfg), ref.run_round(ws, cfg)
    for k in x:
        if isinstance(x[k], np.ndarray):
            assert np.array_equal(x[k], y[k]), k
        else:
            assert x[k] == y[k], k


# ------------------------------------- 4. reference property tests on the port
def test_fused_equals_unfused_port(port):
    """proj/tests/test_codec.cpp:118-140"""
    cc = port.codec()
    w = np.array([8, 4, 4, 2], np.uint8)
    rng = np.random.default_rng(0)
    for trial in range(30):
        base = (rng.standard_normal(1024) * 3).astype(np.float32)
        local = rng.standard_normal(1024).astype(np.float32)
        inc = port.compress_chunk(base, w, cc, port.qctx(trial, 0, 0, 0, 4, True))
        hop = port.qctx(trial, 0, 0, 1, 4, True)
        fused = port.dar_chunk(inc, local, cc, hop)
        unfused = port.compress_chunk(port.decompress_chunk(inc, cc, 1024) + local, w, cc, hop)
        assert fused == unfused


def test_wire_sizes_port(port):
    """proj/tests/test_codec.cpp:142-155"""
    assert port.compressed_size_bits([4]) - 192 == 1168
    assert port.compressed_size_bits([16]) - 192 == 256 * 16
    assert port.compressed_size_bits([]) == 192


def test_correlated_partition_port(port):
    """proj/tests/test_random.cpp:86-106: one slot per 1/n interval"""
    for n in (2, 3, 4, 8, 16):
        for trial in range(50):
            cells = sorted(int(port.correlated_uniform(3, 2, 1, 9, trial, 7, s, n) * n) for s in range(n))
            assert cells == list(range(n))


def test_malformed_rejected_port(port):
    """proj/tests/test_codec.cpp:180-223 (port parser)"""
    cc = port.codec()
    w = np.array([4, 2], np.uint8)
    v = det_values(9, 512)
    b = port.compress_chunk(v, w, cc, port.qctx(9))
    for cut in (1, len(b) // 2, len(b) - 1):
        with pytest.raises(OracleError):
            port.decompress_chunk(b[:cut], cc, 512)
    with pytest.raises(OracleError):
        port.decompress_chunk(b + b"\0", cc, 512)
    t = bytearray(b)
    t[8] += 1
    with pytest.raises(OracleError):
        port.decompress_chunk(bytes(t), cc, 512)
