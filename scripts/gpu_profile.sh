# ncu evidence for profiles/: launch list of a short bench run + one full
# capture of the production mover (k_push_quad), plus the A/B of mover paths.
OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; tail -2 $OUT/pytest_gpu.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 6 --warmup 4 --no-cpu-baseline > $OUT/bench_under_ncu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push_quad -s 6 -c 1 \
  -o $OUT/push_quad python bench.py --steps 4 --warmup 4 --no-cpu-baseline > $OUT/ncu_full.txt 2>&1
tail -2 $OUT/ncu_full.txt
for v in "PB_PUSH_PATH=quad" "PB_PUSH_PATH=tma" "PB_PUSH_PATH=ldg"; do
  env $v timeout 300 python bench.py --steps 40 --warmup 6 --no-cpu-baseline > $OUT/ab_$v.txt 2>&1
done
