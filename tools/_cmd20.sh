python -m pytest tests -m gpu -x -q > gpurun_out/r2_t_bf.log 2>&1; echo T=$?; tail -2 gpurun_out/r2_t_bf.log
for rep in 1 2; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bf4_$rep.json 2>&1
  python bench.py --steps 10 --warmup 3 --n-sim 8 --no-cpu-baseline --no-e2e > gpurun_out/r2_bf8_$rep.json 2>&1
done
echo done
