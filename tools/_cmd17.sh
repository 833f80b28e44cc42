python -m pytest tests -m gpu -x -q > gpurun_out/r2_t_div.log 2>&1; echo T=$?; tail -2 gpurun_out/r2_t_div.log
for v in main heavy0 heavy7; do
  if [ $v = main ]; then unset DQ_LIB_VARIANT; else export DQ_LIB_VARIANT=$v; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_b4_$v.json 2>&1
  python bench.py --steps 10 --warmup 3 --n-sim 8 --no-cpu-baseline --no-e2e > gpurun_out/r2_b8_$v.json 2>&1
done
echo done
