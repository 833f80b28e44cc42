"""DDP comm hook: three DDP steps with the non-blocking dynamiq_hook.

Every bucket's hooked gradient is bit-identical to dq.run_round over the gathered per-rank
buckets (same SharedSeed round) / world; ranks agree; the result is close to DDP's NCCL
mean.  Runs tools/ddp_check.py under torchrun on every visible GPU (>= 2)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ddp_hook_bit_exact_and_non_blocking():
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 8)}",
           "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(ROOT, "tools", "ddp_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-2000:] + r.stderr[-2000:]
    res = json.loads(lines[-1])
    assert res["ok"], json.dumps(res)
    assert res["buckets"] >= 3 and all(res["bit_exact_vs_sim_round"])
