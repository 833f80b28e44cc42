#!/bin/bash
# One-GPU measurement pass of round 2 (run under gpurun from the repo root): bench lines,
# the decode-write microbenchmark, compute-sanitizer on small rounds, ncu launch list and
# --set full captures of the hot kernels (exported to CSV on the box: the reports are large).
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/r2m_bench.json 2> $O/r2m_bench.err; echo "bench rc=$?"
python bench.py --steps 10 --warmup 3 --n-sim 8 --no-cpu-baseline --no-e2e > $O/r2m_bench_n8.json 2> $O/r2m_bench_n8.err; echo "bench n8 rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $O/r2m_bench_ref.json 2> $O/r2m_bench_ref.err; echo "ref rc=$?"
./tools/_mb_scatter > $O/r2m_mb_scatter.txt 2>&1; echo "mb rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_round.py > $O/r2m_sanitize_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2m_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/r2m_ncu_launches.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_quant|k_gather|k_stats" -s 17 -c 5 -o /tmp/r2m \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/r2m_ncu_full.log 2>&1; echo "ncu full rc=$?"
tools/ncu_export.sh /tmp/r2m.ncu-rep $O/r2m
ls -la $O
