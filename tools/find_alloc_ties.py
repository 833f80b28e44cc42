#!/usr/bin/env python3
"""Search seeds where the exact-arithmetic plateau crossing differs from the reference's
float-threshold bisection (allocate_fast): python tools/find_alloc_ties.py START STOP.
Found seed 5 at T = 2^22 (used by tests/test_gpu_alloc.py)."""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle.oracle import Oracle
port = Oracle("port")
alpha = 4.0 / np.log2(512.0 / 17.0)
def exact_choice(F, b=4.0, S=256):
    T = F.size
    bbar = b - (8/16 + 16/256)
    budget = T * S * bbar
    pos = F[F > 0].astype(np.float64)
    l = alpha * np.log2(pos)
    flips = np.concatenate([4.0 - l, 8.0 - l]); wts = np.concatenate([np.full(l.size, 2), np.full(l.size, 4)])
    order = np.argsort(flips, kind='stable'); flips = flips[order]; wts = wts[order]
    uf, idx = np.unique(flips, return_index=True)
    cw = np.add.reduceat(wts, idx).cumsum()
    W = int(np.floor(budget / S)) - 2 * T
    while S * (2 * T + W + 1) <= budget: W += 1
    while W >= 0 and S * (2 * T + W) > budget: W -= 1
    L = int(np.searchsorted(cw, W, side='right'))  # first flip with cumulative > W
    if L >= uf.size: u = uf[-1] + 1
    elif L == 0: u = uf[0] - 1
    else: u = 0.5 * (uf[L - 1] + uf[L])
    return u
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(seed)
    T = 1 << 22
    F = (np.exp(8 * rng.standard_normal(T)) * 256).astype(np.float32)
    ue = exact_choice(F)
    w, p, u, pay = port.allocate_fast(F, 4.0)
    if u != ue:
        print("MISMATCH seed", seed, u, ue, flush=True)
    else:
        print("same", seed, flush=True)
