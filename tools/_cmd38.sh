cd /root/repo
export DQ_WAIT_TIMEOUT_S=120
for ns in 0 1; do
DQ_NO_SMALL_ALLOC=$ns timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2983$ns tools/sweep.py --sizes 18:21 --steps 20 > gpurun_out/r2_sweep4_nosmall$ns.jsonl 2>/dev/null; echo S$ns=$?
DQ_NO_SMALL_ALLOC=$ns CUDA_VISIBLE_DEVICES=0 python tools/host_overhead.py > gpurun_out/r2_host_nosmall$ns.jsonl 2>&1
done
