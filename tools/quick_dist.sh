#!/bin/bash
# Quick distributed check on a 4-GPU box: dist_check N=4/N=3 (peer transport), the
# distributed GPU tests, bench.py N=4 ring.  Outputs under gpurun_out/qd/.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/qd
mkdir -p $O
DIST_CHECK_TRANSPORTS=peer timeout 600 $R --nproc-per-node 4 --master-port 29731 tools/dist_check.py > $O/dist4.log 2>&1; echo "dist4 rc=$? $(tail -1 $O/dist4.log | cut -c1-60)"
DIST_CHECK_TRANSPORTS=peer timeout 600 $R --nproc-per-node 3 --master-port 29732 tools/dist_check.py > $O/dist3.log 2>&1; echo "dist3 rc=$? $(tail -1 $O/dist3.log | cut -c1-60)"
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
timeout 600 $R --nproc-per-node 4 --master-port 29733 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"
for f in $O/bench*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], {k: v['ms_per_step'] for k, v in d.get('kernels', {}).items()})" 2>/dev/null; done
