# ncu evidence for profiles/: launch list of a short bench run + one full
# capture of the production mover (k_push_split for config 2) inside the bench, then the
# round-end style checks (tests, smoke, default bench, reference arm).
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 6 --warmup 4 --no-cpu-baseline > $OUT/bench_under_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push_ -s 8 -c 1 \
  -o $OUT/push_mover python bench.py --steps 8 --warmup 4 --no-cpu-baseline > $OUT/ncu_full.txt 2>&1
tail -2 $OUT/ncu_full.txt
bash scripts/gpu_round.sh
