#!/bin/bash
# Full verification batch on a 4-GPU box: GPU test suite, distributed parity at N=2/3/4
# (both transports), then bench.py at N=1/2/4.  Outputs under gpurun_out/vb/.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/vb
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest_gpu.log)"
timeout 600 $R --nproc-per-node 4 --master-port 29701 tools/dist_check.py > $O/dist4.log 2>&1; echo "dist4 rc=$? $(tail -1 $O/dist4.log | cut -c1-200)"
DIST_CHECK_TRANSPORTS=peer timeout 600 $R --nproc-per-node 3 --master-port 29702 tools/dist_check.py > $O/dist3.log 2>&1; echo "dist3 rc=$? $(tail -1 $O/dist3.log | cut -c1-200)"
DIST_CHECK_TRANSPORTS=peer timeout 600 $R --nproc-per-node 2 --master-port 29703 tools/dist_check.py > $O/dist2.log 2>&1; echo "dist2 rc=$? $(tail -1 $O/dist2.log | cut -c1-200)"
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench1.json 2> $O/bench1.err; echo "bench1 rc=$?"
timeout 600 $R --nproc-per-node 2 --master-port 29704 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?"
timeout 600 $R --nproc-per-node 4 --master-port 29705 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"
timeout 600 $R --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --steps 20 --warmup 5 --topology butterfly --no-e2e > $O/bench4_bfly.json 2> $O/bench4_bfly.err; echo "bench4 butterfly rc=$?"
for f in $O/bench*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], {k: v['ms_per_step'] for k, v in d.get('kernels', {}).items()})" 2>/dev/null; done
