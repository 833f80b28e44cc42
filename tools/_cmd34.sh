cd /root/repo
export DQ_WAIT_TIMEOUT_S=60
SIZES=65536,262144,4194304 ITERS=2 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 tools/early_repro.py > gpurun_out/r2_repro_fused.log 2>&1; echo R=$?; grep -c "ok=True" gpurun_out/r2_repro_fused.log
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ddp.py tests/test_gpu_async.py -x -q > gpurun_out/r2_t_fused.log 2>&1; echo T=$?; tail -2 gpurun_out/r2_t_fused.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29802 tools/sweep.py --sizes 16:28:2 > gpurun_out/r2_sweep4_fused.jsonl 2> gpurun_out/r2_sweep4_fused.err; echo S=$?
DIST_GRAPH_SIZES=262144,1048576,4194304 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29803 tools/dist_graph.py > gpurun_out/r2_graph4_fused.json 2> gpurun_out/r2_graph4_fused.err; echo G=$?
