cd /root/repo
python tools/host_overhead.py > gpurun_out/r2_host_sim.jsonl 2>&1; echo H1=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29731 tools/host_overhead.py > gpurun_out/r2_host_n4.jsonl 2> gpurun_out/r2_host_n4.err; echo H4=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_t_all_final4.log 2>&1; echo T=$?; tail -3 gpurun_out/r2_t_all_final4.log
