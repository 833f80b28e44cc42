for rep in 1 2; do
for g in wave legacy; do
  if [ $g = legacy ]; then export DQ_HOP_GRID=legacy; else unset DQ_HOP_GRID; fi
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ab4_${g}_$rep.json 2>&1
  python bench.py --steps 10 --warmup 3 --n-sim 8 --no-cpu-baseline --no-e2e > gpurun_out/r2_ab8_${g}_$rep.json 2>&1
done
done
echo done
