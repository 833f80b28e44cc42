cd /root/repo
DQ_DEBUG_ALLOC=1 timeout 300 python tools/dbg_alloc.py 2 268435456 > gpurun_out/r2_dbg_alloc.log 2>&1; echo DBG=$?
timeout 1200 python -m pytest tests/test_gpu_async.py -x -q -s > gpurun_out/r2_t_async.log 2>&1; echo TA=$?; tail -3 gpurun_out/r2_t_async.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_t_all1.log 2>&1; echo T=$?; tail -3 gpurun_out/r2_t_all1.log
