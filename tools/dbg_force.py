import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2602_08923_b200 as dq
from paper_2602_08923_b200._lib import check, lib
from oracle.oracle import Oracle
port = Oracle("port")
for (n, b, d, seed) in [(8, 4.0, 1 << 15, 31), (4, 4.0, 1 << 16, 27), (8, 4.0, 1 << 15, 5)]:
    ws = [port.generate_worker(d, seed=seed, sigma_log=4.0, rank=r) for r in range(n)]
    want = port.run_round(ws, port.round_cfg(n, b, "ring", seed=1))
    cfg = dq.PipelineConfig(n_workers=n, budget_bits=b, seed=dq.SharedSeed(1, 0))
    for force in (0, 1):
        check(lib().dq_debug_force_host_alloc(force))
        got = dq.run_round([torch.from_numpy(w).cuda() for w in ws], cfg, with_allocation=True)
        s = got.synced.cpu().numpy()
        print(n, b, d, "force", force, "synced", np.array_equal(s.view(np.uint32), want["synced"].view(np.uint32)),
              "widths", np.array_equal(got.widths, want["widths"]), "perm", np.array_equal(got.permutation, want["perm"]),
              "u", got.u, want["u"], "pay", got.payload_bits, want["payload_bits"], "n842", got.info["n8"], got.info["n4"], got.info["n2"])
        if not np.array_equal(s.view(np.uint32), want["synced"].view(np.uint32)):
            bad = np.nonzero(s.view(np.uint32) != want["synced"].view(np.uint32))[0]
            print("  mismatches", bad.size, "first", bad[:10], "sgs", np.unique(bad // 256)[:20])
    check(lib().dq_debug_force_host_alloc(0))
