"""ctypes wrapper over the CPU oracle libraries (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module — as the checker, never as
the thing measured or shipped.  The product package ``paper_2602_08923_b200``
never imports it.

Two implementations share one interface (``oracle/dq_oracle.h``):

* ``Oracle("port")``      -> ``oracle/build/libdqoracle.so`` (plain-C restatement)
* ``Oracle("reference")`` -> ``oracle/_ref/libdqref.so`` (the reference library
  itself, compiled from /root/reference/proj/src by ``oracle/Makefile``)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": (os.path.join(HERE, "build", "libdqoracle.so"), "dqo_"),
    "reference": (os.path.join(HERE, "_ref", "libdqref.so"), "dqref_"),
}

ENTRY_QUANT, SCALE_QUANT, PERMUTATION = 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class QCtx(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("round", C.c_uint64), ("chunk", C.c_uint32),
                ("slot", C.c_uint32), ("n_slots", C.c_uint32), ("correlated", C.c_int32)]


class Codec(C.Structure):
    _fields_ = [("group_size", C.c_uint32), ("super_group_size", C.c_uint32),
                ("hierarchical", C.c_int32), ("non_uniform", C.c_int32)]


class RoundCfg(C.Structure):
    _fields_ = [("n_workers", C.c_uint32), ("group_size", C.c_uint32),
                ("super_group_size", C.c_uint32), ("budget_bits", C.c_double),
                ("non_uniform", C.c_int32), ("variable_width", C.c_int32),
                ("hierarchical", C.c_int32), ("correlated", C.c_int32),
                ("fixed_width", C.c_int32), ("allocator", C.c_int32), ("topology", C.c_int32),
                ("codec", C.c_int32), ("seed", C.c_uint64), ("round", C.c_uint64),
                ("threads", C.c_uint32)]


class RoundOut(C.Structure):
    _fields_ = [("wire_hash", C.c_uint64), ("vnmse", C.c_double), ("mse", C.c_double),
                ("u", C.c_double), ("payload_bits", C.c_uint64), ("stats_bits", C.c_uint64),
                ("wire_payload_bits", C.c_uint64), ("scale_bits", C.c_uint64),
                ("header_bits", C.c_uint64), ("repr_bits", C.c_uint64),
                ("compressed_coordinates", C.c_uint64), ("transmitted_coordinates", C.c_uint64)]


def build() -> None:
    """Compile the restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind][0])


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


class Oracle:
    def __init__(self, kind: str = "port"):
        path, prefix = PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.pre = prefix
        f = self._f
        u64, u32, i32, dbl, sz = C.c_uint64, C.c_uint32, C.c_int, C.c_double, C.c_size_t
        P = C.POINTER
        f("random_bits", u64, [u64, u64, u32, u64, u64, u64])
        f("uniform_at", dbl, [u64, u64, u32, u64, u64, u64])
        f("permutation_slot", i32, [u64, u64, u32, u64, u64, u64, u32, u32, P(u32)])
        f("correlated_uniform", i32, [u64, u64, u32, u64, u64, u64, u32, u32, P(dbl)])
        f("codebook", i32, [i32, i32, P(C.c_float)])
        f("compressed_size_bits", u64, [P(C.c_uint8), sz, u32, u32, i32])
        f("compress_chunk", i32, [P(C.c_float), P(C.c_uint8), sz, P(Codec), P(QCtx), u32,
                                  P(C.c_uint8), sz, P(sz)])
        f("dar_chunk", i32, [P(C.c_uint8), sz, P(C.c_float), sz, P(Codec), P(QCtx), u32,
                             P(C.c_uint8), sz, P(sz)])
        f("decompress_chunk", i32, [P(C.c_uint8), sz, P(Codec), P(C.c_float), sz])
        f("decompress_accumulate", i32, [P(C.c_uint8), sz, P(Codec), P(C.c_float), sz])
        f("compute_stats", i32, [P(C.c_float), sz, u32, u32, P(C.c_float), P(C.c_float)])
        f("reduce_stats", i32, [P(C.c_float), P(C.c_float), u32, sz, P(C.c_float), P(C.c_float)])
        f("allocate_fast", i32, [P(C.c_float), sz, dbl, u32, u32, i32, P(C.c_uint8), P(u32),
                                 P(dbl), P(u64)])
        f("allocate_general", i32, [P(C.c_float), sz, dbl, u32, u32, i32, P(i32), i32, P(C.c_uint8),
                                    P(u32), P(dbl), P(u64)])
        f("allocate_fast_stateful", i32, [P(C.c_float), sz, dbl, u32, u32, i32, P(dbl), P(C.c_uint8),
                                          P(u32), P(dbl), P(u64)])
        f("build_permutation", i32, [P(C.c_uint8), sz, P(u32)])
        f("schedule", i32, [u32, i32, u32, P(u32), u32, P(u32), P(u32), P(u32), P(u32)])
        f("run_round", i32, [P(P(C.c_float)), sz, P(RoundCfg), P(C.c_float), P(C.c_uint8),
                             P(u32), P(RoundOut)])
        f("generate_worker", i32, [i32, sz, u64, dbl, u32, u32, P(C.c_float)])
        f("last_error", C.c_char_p, [])

    def _f(self, name, restype, argtypes):
        fn = getattr(self.lib, self.pre + name)
        fn.restype = restype
        fn.argtypes = argtypes
        setattr(self, "_" + name, fn)

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self._last_error().decode())

    # ---- PRNG
    def random_bits(self, seed, rnd, purpose, chunk, sg, entry) -> int:
        return self._random_bits(seed, rnd, purpose, chunk, sg, entry)

    def uniform_at(self, seed, rnd, purpose, chunk, sg, entry) -> float:
        return self._uniform_at(seed, rnd, purpose, chunk, sg, entry)

    def permutation_slot(self, seed, rnd, purpose, chunk, sg, entry, slot, n) -> int:
        out = C.c_uint32()
        self._check(self._permutation_slot(seed, rnd, purpose, chunk, sg, entry, slot, n, C.byref(out)))
        return out.value

    def correlated_uniform(self, seed, rnd, purpose, chunk, sg, entry, slot, n) -> float:
        out = C.c_double()
        self._check(self._correlated_uniform(seed, rnd, purpose, chunk, sg, entry, slot, n, C.byref(out)))
        return out.value

    def codebook(self, width: int, non_uniform: bool = True) -> np.ndarray:
        out = np.zeros(1 << (width - 1), np.float32)
        self._check(self._codebook(width, int(non_uniform), _p(out, C.c_float)))
        return out

    # ---- codec (reference wire bytes)
    def compressed_size_bits(self, widths, S=256, s=16, hierarchical=True) -> int:
        w = np.ascontiguousarray(widths, np.uint8)
        return self._compressed_size_bits(_p(w, C.c_uint8), w.size, S, s, int(hierarchical))

    @staticmethod
    def codec(s=16, S=256, hierarchical=True, non_uniform=True) -> Codec:
        return Codec(s, S, int(hierarchical), int(non_uniform))

    @staticmethod
    def qctx(seed=1, rnd=0, chunk=0, slot=0, n_slots=1, correlated=True) -> QCtx:
        return QCtx(seed, rnd, chunk, slot, n_slots, int(correlated))

    def compress_chunk(self, values, widths, codec: Codec, q: QCtx, first_sg=0) -> bytes:
        v = np.ascontiguousarray(values, np.float32)
        w = np.ascontiguousarray(widths, np.uint8)
        cap = self.compressed_size_bits(w, codec.super_group_size, codec.group_size,
                                        codec.hierarchical) // 8
        out = np.zeros(max(cap, 1), np.uint8)
        n = C.c_size_t()
        self._check(self._compress_chunk(_p(v, C.c_float), _p(w, C.c_uint8), w.size, C.byref(codec),
                                         C.byref(q), first_sg, _p(out, C.c_uint8), out.size, C.byref(n)))
        return out[: n.value].tobytes()

    def dar_chunk(self, chunk: bytes, local, codec: Codec, q: QCtx, first_sg=0) -> bytes:
        b = np.frombuffer(chunk, np.uint8).copy()
        loc = np.ascontiguousarray(local, np.float32)
        out = np.zeros(max(b.size, 1), np.uint8)
        n = C.c_size_t()
        self._check(self._dar_chunk(_p(b, C.c_uint8), b.size, _p(loc, C.c_float), loc.size,
                                    C.byref(codec), C.byref(q), first_sg, _p(out, C.c_uint8),
                                    out.size, C.byref(n)))
        return out[: n.value].tobytes()

    def decompress_chunk(self, chunk: bytes, codec: Codec, n_out: int) -> np.ndarray:
        b = np.frombuffer(chunk, np.uint8).copy()
        out = np.zeros(n_out, np.float32)
        self._check(self._decompress_chunk(_p(b, C.c_uint8), b.size, C.byref(codec),
                                           _p(out, C.c_float), n_out))
        return out

    def decompress_accumulate(self, chunk: bytes, codec: Codec, acc: np.ndarray) -> np.ndarray:
        b = np.frombuffer(chunk, np.uint8).copy()
        a = np.ascontiguousarray(acc, np.float32).copy()
        self._check(self._decompress_accumulate(_p(b, C.c_uint8), b.size, C.byref(codec),
                                                _p(a, C.c_float), a.size))
        return a

    # ---- stats / allocation
    def compute_stats(self, x, s=16, S=256):
        v = np.ascontiguousarray(x, np.float32)
        nsg = (v.size + S - 1) // S
        m = np.zeros(nsg, np.float32)
        q = np.zeros(nsg, np.float32)
        self._check(self._compute_stats(_p(v, C.c_float), v.size, s, S, _p(m, C.c_float), _p(q, C.c_float)))
        return m, q

    def reduce_stats(self, means, sqs):
        m = np.ascontiguousarray(means, np.float32)
        q = np.ascontiguousarray(sqs, np.float32)
        n, nsg = m.shape
        gm = np.zeros(nsg, np.float32)
        gq = np.zeros(nsg, np.float32)
        self._check(self._reduce_stats(_p(m, C.c_float), _p(q, C.c_float), n, nsg,
                                       _p(gm, C.c_float), _p(gq, C.c_float)))
        return gm, gq

    def allocate_fast(self, F, budget_bits, s=16, S=256, hierarchical=True):
        f = np.ascontiguousarray(F, np.float32)
        w = np.zeros(max(f.size, 1), np.uint8)
        p = np.zeros(max(f.size, 1), np.uint32)
        u = C.c_double()
        pay = C.c_uint64()
        self._check(self._allocate_fast(_p(f, C.c_float), f.size, budget_bits, s, S, int(hierarchical),
                                        _p(w, C.c_uint8), _p(p, C.c_uint32), C.byref(u), C.byref(pay)))
        return w[: f.size], p[: f.size], u.value, pay.value

    def allocate_general(self, F, budget_bits, widths=(2, 4, 8), s=16, S=256, hierarchical=True):
        """proj/src/allocation.cpp:121-168 -> (widths, permutation, u = resolved base threshold, payload)"""
        f = np.ascontiguousarray(F, np.float32)
        W = np.ascontiguousarray(widths, np.int32)
        w = np.zeros(max(f.size, 1), np.uint8)
        p = np.zeros(max(f.size, 1), np.uint32)
        u = C.c_double()
        pay = C.c_uint64()
        self._check(self._allocate_general(_p(f, C.c_float), f.size, budget_bits, s, S, int(hierarchical),
                                           _p(W, C.c_int), W.size, _p(w, C.c_uint8), _p(p, C.c_uint32),
                                           C.byref(u), C.byref(pay)))
        return w[: f.size], p[: f.size], u.value, pay.value

    def allocate_fast_stateful(self, F, budget_bits, state, s=16, S=256, hierarchical=True):
        """proj/src/allocation.cpp:262-300; state = [lo, hi, u] (FastAllocatorState) ->
        (widths, permutation, u used this round, payload, next state)"""
        f = np.ascontiguousarray(F, np.float32)
        st = np.array(state, np.float64)
        w = np.zeros(max(f.size, 1), np.uint8)
        p = np.zeros(max(f.size, 1), np.uint32)
        u = C.c_double()
        pay = C.c_uint64()
        self._check(self._allocate_fast_stateful(_p(f, C.c_float), f.size, budget_bits, s, S, int(hierarchical),
                                                 _p(st, C.c_double), _p(w, C.c_uint8), _p(p, C.c_uint32),
                                                 C.byref(u), C.byref(pay)))
        return w[: f.size], p[: f.size], u.value, pay.value, [float(x) for x in st]

    def build_permutation(self, widths):
        w = np.ascontiguousarray(widths, np.uint8)
        p = np.zeros(max(w.size, 1), np.uint32)
        self._check(self._build_permutation(_p(w, C.c_uint8), w.size, _p(p, C.c_uint32)))
        return p[: w.size]

    def schedule(self, n, topology, chunk):
        """topology.cpp:8-70 -> (events [(sender, receiver, slot)], sink_slot, n_slots, n_gather)"""
        ev = np.zeros(3 * 64 * 8, np.uint32)
        ne, ss, ns, ng = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        self._check(self._schedule(n, {"ring": 0, "butterfly": 1}[topology], chunk, _p(ev, C.c_uint32), 64 * 8,
                                   C.byref(ne), C.byref(ss), C.byref(ns), C.byref(ng)))
        return [tuple(int(x) for x in ev[3 * e:3 * e + 3]) for e in range(ne.value)], ss.value, ns.value, ng.value

    # ---- engine
    @staticmethod
    def round_cfg(n_workers=4, budget_bits=5.0, topology="ring", seed=1, rnd=0, s=16, S=256,
                  non_uniform=True, variable_width=True, hierarchical=True, correlated=True,
                  fixed_width=4, allocator=None, codec="quantized", threads=1) -> RoundCfg:
        if allocator is None:
            allocator = "fast" if variable_width else "fixed"
        return RoundCfg(n_workers, s, S, budget_bits, int(non_uniform), int(variable_width),
                        int(hierarchical), int(correlated), fixed_width,
                        {"general": 0, "fast": 1, "fixed": 2}[allocator],
                        {"ring": 0, "butterfly": 1}[topology],
                        {"quantized": 0, "lossless": 1}[codec], seed, rnd, threads)

    def run_round(self, workers, cfg: RoundCfg):
        ws = [np.ascontiguousarray(w, np.float32) for w in workers]
        d = ws[0].size
        arr = (C.POINTER(C.c_float) * len(ws))(*[_p(w, C.c_float) for w in ws])
        synced = np.zeros(d, np.float32)
        nsg = (d + cfg.super_group_size - 1) // cfg.super_group_size
        widths = np.zeros(nsg, np.uint8)
        perm = np.zeros(nsg, np.uint32)
        out = RoundOut()
        self._check(self._run_round(arr, d, C.byref(cfg), _p(synced, C.c_float), _p(widths, C.c_uint8),
                                    _p(perm, C.c_uint32), C.byref(out)))
        res = {k: getattr(out, k) for k, _ in RoundOut._fields_}
        res.update(synced=synced, widths=widths, perm=perm)
        return res

    def generate_worker(self, d, seed=1, sigma_log=4.0, rank=0, kind="locality", S=256):
        out = np.zeros(d, np.float32)
        self._check(self._generate_worker(0 if kind == "iid" else 1, d, seed, sigma_log, S, rank,
                                          _p(out, C.c_float)))
        return out
