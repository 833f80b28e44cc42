#!/usr/bin/env python3
"""Device cost of the fused codec kernels per super-group width (one GPU).

Chunks are width-sorted (8-bit super-groups first), so ring chunks differ in cost;
this measures compress / DAR ms per 2^18 super-groups for uniform-width chunks.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_08923_b200 as dq  # noqa: E402


def main():
    nsg = 1 << 18
    g = torch.Generator(device="cuda").manual_seed(1)
    scale = torch.exp(4 * torch.randn(nsg, device="cuda", generator=g))
    x = (torch.randn(nsg, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1).contiguous()
    y = (torch.randn(nsg, 256, device="cuda", generator=g) * scale[:, None]).reshape(-1).contiguous()
    cfg = dq.CodecConfig()
    res = {}
    for w in (8, 4, 2):
        widths = [w] * nsg
        q = dq.QuantContext(dq.SharedSeed(1, 0), chunk_index=1, hop_slot=0, n_slots=4)
        ch = dq.compress_chunk(x, widths, cfg, q)
        q1 = dq.QuantContext(dq.SharedSeed(1, 0), chunk_index=1, hop_slot=1, n_slots=4)
        for name, fn in (("compress", lambda: dq.compress_chunk(x, widths, cfg, q)),
                         ("dar", lambda: dq.decompress_accumulate_recompress(ch, y, cfg, q1))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                fn()
            b.record()
            torch.cuda.synchronize()
            res[f"{name}_w{w}_ms"] = round(a.elapsed_time(b) / 10, 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
