cd /root/repo
python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/r2_t_dist26.log 2>&1; echo T=$?; tail -2 gpurun_out/r2_t_dist26.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29721 tools/sweep.py --sizes 18:30 > gpurun_out/r2_sweep4b.jsonl 2> gpurun_out/r2_sweep4b.err; echo S4=$?
DIST_GRAPH_SIZES=262144,1048576,4194304 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29722 tools/dist_graph.py > gpurun_out/r2_graph4b.json 2> gpurun_out/r2_graph4b.err; echo G4=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29723 tools/sweep.py --sizes 18:26:2 > gpurun_out/r2_sweep2b.jsonl 2> gpurun_out/r2_sweep2b.err; echo S2=$?
