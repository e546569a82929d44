# per-kernel launch list of the config-3 step (field solve + absorbing + sort)
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/c3_launches.csv \
  python bench.py --workload c3 --steps 6 --warmup 4 --no-cpu-baseline > $OUT/c3_under_ncu.txt 2>&1
for f in 0 1; do
  PB_FUSED_FIELD=$f timeout 600 python bench.py --workload c3 --steps 400 --warmup 10 --no-cpu-baseline > $OUT/c3_fused$f.txt 2>&1
  echo "fused=$f $(tail -1 $OUT/c3_fused$f.txt | cut -c1-200)"
done
