# ncu evidence for the push kernel: launch list + one full capture.
set -x
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push -s 4 -c 1 \
  -o $OUT/push python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.txt 2>&1
ls -la $OUT
