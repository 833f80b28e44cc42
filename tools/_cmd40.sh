cd /root/repo
export DQ_WAIT_TIMEOUT_S=120
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_final2_tests_4gpu.log 2>&1; echo T=$?; tail -2 gpurun_out/r2_final2_tests_4gpu.log
DQ_LIB_VARIANT=debug timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_final2_debug_4gpu.log 2>&1; echo D=$?; tail -2 gpurun_out/r2_final2_debug_4gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final2_smoke.log 2>&1; echo SM=$?; tail -1 gpurun_out/r2_final2_smoke.log
CUDA_VISIBLE_DEVICES=0 python bench.py > gpurun_out/r2_final2_bench_n1.json 2> gpurun_out/r2_final2_bench_n1.err; echo B1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29851 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_final2_bench_n4.json 2> gpurun_out/r2_final2_bench_n4.err; echo B4=$?
