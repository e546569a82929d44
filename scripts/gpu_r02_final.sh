# r02 evidence pass: ncu launch lists (c2, c3) and full captures (c2 mover, c3 mover, c3 field step),
# then the round-end checks (all -m gpu tests, smoke, default bench, reference arm) and one line per workload
OUT=gpurun_out
mkdir -p $OUT
bash scripts/gpu_profile.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_push_ -s 8 -c 1 \
  -o $OUT/push_mover_c3 python bench.py --workload c3 --steps 8 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_fused -s 8 -c 1 \
  -o $OUT/field_fused_c3 python bench.py --workload c3 --steps 8 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv \
  python bench.py --workload c3 --steps 30 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
ls $OUT/*.ncu-rep
for w in c2 c3 c4 c5 c4b; do
  timeout 900 python bench.py --workload $w --steps 400 --warmup 10 --no-cpu-baseline > $OUT/wl_$w.txt 2>&1
  tail -1 $OUT/wl_$w.txt | cut -c1-200
done
