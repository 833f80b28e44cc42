cd /root/repo
export DQ_WAIT_TIMEOUT_S=120
DQ_LIB_VARIANT=debug timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_final_debug_checks_4gpu.log 2>&1; echo D=$?; tail -3 gpurun_out/r2_final_debug_checks_4gpu.log
