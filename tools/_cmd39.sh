cd /root/repo
export DQ_WAIT_TIMEOUT_S=120
CUDA_VISIBLE_DEVICES=0 DQ_LIB_VARIANT=phases python tools/small_phases.py > gpurun_out/r2_small_phases6.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_async.py tests/test_gpu_round.py tests/test_gpu_dist.py -x -q > gpurun_out/r2_t_probe.log 2>&1; echo T=$?; tail -2 gpurun_out/r2_t_probe.log
CUDA_VISIBLE_DEVICES=0 timeout 400 python tools/fuzz_rounds.py --seconds 200 --seed 92 > gpurun_out/r2_fuzz_probe.log 2>&1; echo F=$?; tail -1 gpurun_out/r2_fuzz_probe.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29841 tools/sweep.py --sizes 16:22 --steps 20 > gpurun_out/r2_sweep4_probe.jsonl 2>/dev/null; echo S=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29842 tools/dist_fuzz.py --iters 400 --seed 93 > gpurun_out/r2_dist_fuzz_probe.log 2>&1; echo DF=$?; grep '"world"' gpurun_out/r2_dist_fuzz_probe.log | tail -1
