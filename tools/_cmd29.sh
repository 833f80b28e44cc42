cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_round.py tests/test_gpu_async.py tests/test_gpu_dist.py tests/test_gpu_ddp.py tests/test_gpu_configs.py -x -q > gpurun_out/r2_t_pdl.log 2>&1; echo T=$?; tail -3 gpurun_out/r2_t_pdl.log
for pdl in 1 0; do
DQ_PDL=$pdl python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2974$pdl tools/sweep.py --sizes 16:28:2 > gpurun_out/r2_sweep4_pdl$pdl.jsonl 2> gpurun_out/r2_sweep4_pdl$pdl.err; echo S$pdl=$?
DQ_PDL=$pdl CUDA_VISIBLE_DEVICES=0 python bench.py --steps 30 --warmup 5 --no-e2e > gpurun_out/r2_bench_n1_pdl$pdl.json 2> gpurun_out/r2_bench_n1_pdl$pdl.err; echo B$pdl=$?
DQ_PDL=$pdl CUDA_VISIBLE_DEVICES=0 python tools/host_overhead.py > gpurun_out/r2_host_sim_pdl$pdl.jsonl 2>&1
done
DIST_GRAPH_SIZES=262144,1048576,4194304 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29752 tools/dist_graph.py > gpurun_out/r2_graph4_pdl.json 2> gpurun_out/r2_graph4_pdl.err; echo G4=$?
