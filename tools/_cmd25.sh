cd /root/repo
python bench.py > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo B1=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_n1.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2_launches_n1.log 2>&1; echo L1=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_launches_small.csv python tools/profile_round.py 262144 4 3 > gpurun_out/r2_launches_small.log 2>&1; echo LS=$?
ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/r2_round_full python tools/profile_round.py 67108864 4 1 > gpurun_out/r2_round_full.log 2>&1; echo NF=$?
bash tools/ncu_export.sh gpurun_out/r2_round_full.ncu-rep gpurun_out/r2_round_full; echo EX=$?
ls -la gpurun_out | tail -5
DQ_LIB_VARIANT=debug timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/r2_debug_checks.log 2>&1; echo DBG=$?; tail -3 gpurun_out/r2_debug_checks.log
