cd /root/repo
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29771 tools/dist_fuzz.py --iters 1500 --seed 123 > gpurun_out/r2_dist_fuzz_final.log 2>&1; echo DF=$?; grep '"world"' gpurun_out/r2_dist_fuzz_final.log | tail -1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29772 tools/dist_fuzz.py --iters 400 --seed 124 > gpurun_out/r2_dist_fuzz_final3.log 2>&1; echo DF3=$?; grep '"world"' gpurun_out/r2_dist_fuzz_final3.log | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 500 python tools/fuzz_rounds.py --seconds 360 --seed 81 > gpurun_out/r2_fuzz_final.log 2>&1; echo F=$?; tail -1 gpurun_out/r2_fuzz_final.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29773 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_bench_n4_final.json 2> gpurun_out/r2_bench_n4_final.err; echo B4=$?
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29774 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_bench_n2_final.json 2> gpurun_out/r2_bench_n2_final.err; echo B2=$?
