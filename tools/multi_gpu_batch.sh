#!/bin/bash
# Multi-GPU measurement batch for profiles/ (run on a 4-GPU box):
# parity at N=3, message-size sweeps per transport, budget/topology sweep, bench at N=2/4.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/mg
mkdir -p $O
DIST_CHECK_TRANSPORTS=peer timeout 600 $R --nproc-per-node 3 --master-port 29601 tools/dist_check.py > $O/dist3.log 2>&1; echo "dist3 rc=$?"
timeout 900 $R --nproc-per-node 4 --master-port 29602 tools/sweep.py --sizes 18:30 --transport peer > $O/sweep4_peer.jsonl 2> $O/sweep4_peer.err; echo "sweep peer rc=$?"
timeout 600 $R --nproc-per-node 4 --master-port 29603 tools/sweep.py --sizes 18:30 --transport nccl > $O/sweep4_nccl.jsonl 2> $O/sweep4_nccl.err; echo "sweep nccl rc=$?"
timeout 600 $R --nproc-per-node 4 --master-port 29604 tools/sweep.py --sizes 26:26 --budgets 2,3,4,6 --topology butterfly,ring > $O/sweep4_budgets.jsonl 2> $O/sweep4_budgets.err; echo "sweep budgets rc=$?"
timeout 600 $R --nproc-per-node 2 --master-port 29605 tools/sweep.py --sizes 18:30 --transport peer > $O/sweep2_peer.jsonl 2> $O/sweep2_peer.err; echo "sweep2 rc=$?"
timeout 600 $R --nproc-per-node 2 --master-port 29606 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?"
timeout 600 $R --nproc-per-node 4 --master-port 29607 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench4.json 2> $O/bench4.err; echo "bench4 rc=$?"
timeout 600 $R --nproc-per-node 4 --master-port 29608 bench.py --gpus 4 --steps 20 --warmup 5 --topology butterfly --no-e2e > $O/bench4_bfly.json 2> $O/bench4_bfly.err; echo "bench4 butterfly rc=$?"
