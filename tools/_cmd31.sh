cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_round.py tests/test_gpu_async.py tests/test_gpu_dist.py tests/test_gpu_ddp.py -x -q > gpurun_out/r2_t_early.log 2>&1; echo T=$?; tail -3 gpurun_out/r2_t_early.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29781 tools/sweep.py --sizes 16:24:2 > gpurun_out/r2_sweep4_early.jsonl 2> gpurun_out/r2_sweep4_early.err; echo S=$?
DIST_GRAPH_SIZES=262144,1048576,4194304 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29782 tools/dist_graph.py > gpurun_out/r2_graph4_early.json 2> gpurun_out/r2_graph4_early.err; echo G=$?
CUDA_VISIBLE_DEVICES=0 python tools/host_overhead.py > gpurun_out/r2_host_sim_early.jsonl 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29783 tools/dist_fuzz.py --iters 400 --seed 322 > gpurun_out/r2_dist_fuzz_early.log 2>&1; echo DF=$?; grep '"world"' gpurun_out/r2_dist_fuzz_early.log | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/fuzz_rounds.py --seconds 150 --seed 83 > gpurun_out/r2_fuzz_early.log 2>&1; echo F=$?; tail -1 gpurun_out/r2_fuzz_early.log
