cd /root/repo
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_t_all_final1.log 2>&1; echo T=$?; tail -3 gpurun_out/r2_t_all_final1.log
DQ_LIB_VARIANT=debug timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_debug_checks2.log 2>&1; echo D=$?; tail -3 gpurun_out/r2_debug_checks2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo SM=$?
python bench.py > gpurun_out/r2_bench_n1_final.json 2> gpurun_out/r2_bench_n1_final.err; echo B1=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref_n1.json 2> gpurun_out/r2_bench_ref_n1.err; echo BR=$?
