cd /root/repo
export DQ_WAIT_TIMEOUT_S=120
CUDA_VISIBLE_DEVICES=0 timeout 800 python tools/fuzz_rounds.py --seconds 600 --seed 2024 > gpurun_out/r2_final_fuzz600.log 2>&1 &
FZ=$!
CUDA_VISIBLE_DEVICES=1,2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29821 tools/dist_fuzz.py --iters 1500 --seed 2025 > gpurun_out/r2_final_dist_fuzz_n2.log 2>&1; echo DF2=$?; grep '"world"' gpurun_out/r2_final_dist_fuzz_n2.log | tail -1
wait $FZ; echo F=$?; tail -1 gpurun_out/r2_final_fuzz600.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29822 tools/dist_fuzz.py --iters 1500 --seed 2026 > gpurun_out/r2_final_dist_fuzz_n4b.log 2>&1; echo DF4=$?; grep '"world"' gpurun_out/r2_final_dist_fuzz_n4b.log | tail -1
