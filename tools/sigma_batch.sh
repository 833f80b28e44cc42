#!/bin/bash
# Input-distribution batch (sigma_log = 4 heavy-tailed, 1 budget-sensitive,
# 0 iid) — bench.py at N=1 and N=4 ring, no e2e leg.  Outputs under gpurun_out/sg/.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/sg
mkdir -p $O
for s in 0 1 4; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --sigma-log $s > $O/n1_s$s.json 2> $O/n1_s$s.err; echo "n1 sigma=$s rc=$?"
  timeout 600 $R --nproc-per-node 4 --master-port 2975$s bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --sigma-log $s > $O/n4_s$s.json 2> $O/n4_s$s.err; echo "n4 sigma=$s rc=$?"
done
for f in $O/*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], d.get('vnmse', d.get('config', {}).get('vnmse')), d.get('config', {}).get('bits_per_entry'))" 2>/dev/null; done
