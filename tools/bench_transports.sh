#!/bin/bash
# N=4 bench with each ring transport (peer memory vs NCCL p2p); per-kernel-family ms/step.
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29530 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench4_peer.json 2> gpurun_out/bench4_peer.err
DQ_TRANSPORT=nccl timeout 300 $R --master-port 29531 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench4_nccl.json 2> gpurun_out/bench4_nccl.err
for t in peer nccl; do tail -1 gpurun_out/bench4_$t.json | python -c "
import sys,json; r=json.loads(sys.stdin.read()); print('$t', r['ms_per_step'], {k:(v['launches'],v['ms_per_step']) for k,v in r['kernels'].items()})"; done
