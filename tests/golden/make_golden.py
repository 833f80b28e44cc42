#!/usr/bin/env python3
"""Generate tests/golden/golden.json from the REFERENCE library (oracle/_ref).

Run in the dev container, where /root/reference exists and oracle/Makefile has
compiled the reference sources into oracle/_ref/libdqref.so:

    make -C oracle && python tests/golden/make_golden.py

Everything here is a function of small deterministic inputs (listed in the
file), so the fixtures are compact: byte strings are stored as hex when short
and as sha256 digests otherwise.  tests/test_oracle.py pins the C restatement
(oracle/build/libdqoracle.so) and the device path against these values.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def f32sha(a: np.ndarray) -> str:
    return sha(np.ascontiguousarray(a, np.float32).tobytes())


def det_values(seed: int, n: int) -> np.ndarray:
    """Inputs from integer arithmetic only (platform independent)."""
    rng = np.random.default_rng(seed)
    mant = rng.integers(-(1 << 23), 1 << 23, n).astype(np.float64)
    expo = rng.integers(-20, 10, n // 256 + 1).repeat(256)[:n].astype(np.float64)
    v = (mant * np.exp2(expo - 23)).astype(np.float32)
    v[rng.integers(0, n, max(1, n // 50))] = 0.0
    return v


def main():
    R = Oracle("reference")
    g = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference library)"}
    g["random_bits"] = [[s, r, p, c, sg, e, R.random_bits(s, r, p, c, sg, e)]
                        for (s, r, p, c, sg, e) in [(1, 0, 1, 0, 0, 0), (1, 0, 3, 2, 5, 7), (123, 7, 2, 3, 5, 9),
                                                    (2**63 + 5, 2**40, 1, 2**31, 2**32 + 1, (9 << 32) | 77)]]
    g["uniform_at"] = [[1, 0, 2, 0, 3, 1 | (2 << 32), R.uniform_at(1, 0, 2, 0, 3, 1 | (2 << 32)).hex()]]
    g["permutation"] = {str(n): [R.permutation_slot(1, 0, 3, 0, 0, 0, s, n) for s in range(n)]
                        for n in (2, 3, 4, 5, 8, 16)}
    g["correlated_uniform"] = [R.correlated_uniform(1, 0, 1, 0, 0, 0, s, 8).hex() for s in range(8)]
    g["codebooks"] = {f"{w}_{u}": [float(x).hex() for x in R.codebook(w, u == "nu")]
                      for w in (2, 4, 8) for u in ("nu", "u")}
    cases = []
    for i, (runs, slot, nsl, corr, nu) in enumerate([((2, 3, 4), 0, 4, True, True), ((1, 0, 5), 3, 4, True, True),
                                                      ((4, 4, 4), 7, 8, True, True), ((3, 3, 3), 2, 3, False, True),
                                                      ((0, 6, 2), 1, 2, True, False), ((5, 1, 1), 9, 16, True, True)]):
        w = np.array([8] * runs[0] + [4] * runs[1] + [2] * runs[2], np.uint8)
        v = det_values(100 + i, w.size * 256)
        loc = det_values(200 + i, w.size * 256)
        cc = R.codec(16, 256, True, nu)
        q0 = R.qctx(1 + i, i, i % 3, slot, nsl, corr)
        comp = R.compress_chunk(v, w, cc, q0, first_sg=17 * i)
        q1 = R.qctx(1 + i, i, i % 3, min(slot + 1, nsl - 1), nsl, corr)
        dar = R.dar_chunk(comp, loc, cc, q1, first_sg=17 * i)
        dec = R.decompress_chunk(comp, cc, v.size)
        da = R.decompress_accumulate(comp, cc, loc)
        cases.append({"seed_values": 100 + i, "seed_local": 200 + i, "runs": runs, "slot": slot, "n_slots": nsl,
                      "correlated": corr, "non_uniform": nu, "seed": 1 + i, "round": i, "chunk": i % 3,
                      "first_sg": 17 * i, "compress_sha": sha(comp), "compress_head": comp[:64].hex(),
                      "dar_slot": min(slot + 1, nsl - 1), "dar_sha": sha(dar), "decompress_sha": f32sha(dec),
                      "da_sha": f32sha(da)})
    g["codec"] = cases
    st = []
    for i, d in enumerate([256, 1000, 4096 + 3]):
        x = det_values(300 + i, d)
        m, q = R.compute_stats(x)
        st.append({"seed": 300 + i, "d": d, "mean_sha": f32sha(m), "sq_sha": f32sha(q)})
    g["stats"] = st
    al = []
    rng = np.random.default_rng(5)
    Fs = {"lognormal": np.exp(8 * rng.standard_normal(3000)).astype(np.float32),
          "zeros_mixed": np.where(rng.random(2000) < 0.2, 0, np.exp(3 * rng.standard_normal(2000))).astype(np.float32),
          "constant": np.full(500, 3.0, np.float32)}
    for name, F in Fs.items():
        for b in (3, 4, 5, 6):
            w, p, u, pay = R.allocate_fast(F, b)
            al.append({"name": name, "b": b, "F_sha": f32sha(F), "widths_sha": sha(w.tobytes()),
                       "perm_sha": sha(p.astype(np.uint32).tobytes()), "u": u.hex(), "payload_bits": pay})
    g["allocation"] = al
    ga = []
    for name, F in Fs.items():
        for W in ((2, 4, 8), (1, 2, 4, 8, 16)):
            for b in (3, 5):
                w, p, u, pay = R.allocate_general(F, b, W)
                ga.append({"name": name, "b": b, "W": list(W), "widths_sha": sha(w.tobytes()),
                           "perm_sha": sha(p.astype(np.uint32).tobytes()), "u": u.hex(), "payload_bits": pay})
    g["allocation_general"] = ga
    g["allocation_inputs"] = {"rng_seed": 5, "note": "F arrays regenerated by the same numpy calls"}
    rounds = []
    for (n, d, b, topo, seed, alloc) in [(4, 1 << 14, 4, "ring", 1, "fast"), (4, (1 << 13) + 77, 5, "ring", 2, "fast"),
                                         (8, 1 << 14, 4, "butterfly", 1, "fast"), (3, 1 << 13, 6, "ring", 3, "fast"),
                                         (2, 1 << 13, 3, "butterfly", 4, "fast"),
                                         (4, 1 << 14, 4, "ring", 5, "general")]:
        ws = [R.generate_worker(d, seed=seed, sigma_log=4.0, rank=r) for r in range(n)]
        res = R.run_round(ws, R.round_cfg(n, b, topo, seed=seed, allocator=alloc))
        rounds.append({"n": n, "d": d, "b": b, "topology": topo, "seed": seed, "allocator": alloc,
                       "inputs_sha": sha(b"".join(w.tobytes() for w in ws)),
                       "wire_hash": f"{res['wire_hash']:016x}", "synced_sha": f32sha(res["synced"]),
                       "widths_sha": sha(res["widths"].tobytes()), "perm_sha": sha(res["perm"].tobytes()),
                       "u": res["u"].hex(), "payload_bits": res["payload_bits"], "vnmse": res["vnmse"].hex()})
    g["rounds"] = rounds
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
