cd /root/repo
export DQ_WAIT_TIMEOUT_S=120
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_final_tests_4gpu.log 2>&1; echo T=$?; tail -3 gpurun_out/r2_final_tests_4gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1; echo SM=$?; tail -1 gpurun_out/r2_final_smoke.log
CUDA_VISIBLE_DEVICES=0 python bench.py > gpurun_out/r2_final_bench_n1.json 2> gpurun_out/r2_final_bench_n1.err; echo B1=$?
CUDA_VISIBLE_DEVICES=0 python bench.py --n-sim 8 --steps 20 --warmup 5 --no-e2e > gpurun_out/r2_final_bench_nsim8.json 2> gpurun_out/r2_final_bench_nsim8.err; echo B8=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_final_bench_n4.json 2> gpurun_out/r2_final_bench_n4.err; echo B4=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_final_bench_n2.json 2> gpurun_out/r2_final_bench_n2.err; echo B2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29813 tools/dist_fuzz.py --iters 800 --seed 777 > gpurun_out/r2_final_dist_fuzz.log 2>&1; echo DF=$?; grep '"world"' gpurun_out/r2_final_dist_fuzz.log | tail -1
CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_final_launches_n1.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2_final_launches_n1.log 2>&1; echo L=$?
