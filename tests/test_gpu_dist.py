"""Multi-GPU parity: dq_allreduce (peer-memory and NCCL ring transports, NCCL butterfly)
== the simulated round == the oracle (bit-exact).

Launches tools/dist_check.py with torchrun on every visible GPU (>= 2 needed)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_distributed_allreduce_matches_simulation():
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "tools", "dist_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], json.dumps(res, indent=1)


def test_back_to_back_async_rounds():
    """24 all-reduces enqueued without host syncs (sizes alternate: region regrowth, epochs,
    round parities) — every output bit-identical to the simulated round and across ranks."""
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tools", "dist_stress.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], json.dumps(res, indent=1)


def test_distributed_allreduce_three_ranks():
    """N = 3 (non-power-of-two slot count: the float-threshold rounding decision, the ring
    permutation slices with n = 3) on the peer transport, against the simulated round."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 3:
        pytest.skip("needs >= 3 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=3",
           "--master-addr=127.0.0.1", "--master-port=29535", os.path.join(ROOT, "tools", "dist_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, DIST_CHECK_TRANSPORTS="peer"))
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], json.dumps(res, indent=1)
    assert res["world"] == 3


def test_distributed_round_in_cuda_graph():
    """dq_allreduce captured in a CUDA graph (device-side epochs and allocation): replays on
    new inputs equal the simulated round and agree across ranks."""
    torch = pytest.importorskip("torch")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29537", os.path.join(ROOT, "tools", "dist_graph.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], json.dumps(res, indent=1)
