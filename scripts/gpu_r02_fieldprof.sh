# r02: config-3 launch list and a full capture of k_field_fused on the final build
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_field_fused -s 8 -c 1 \
  -o $OUT/field_fused_c3_final python bench.py --workload c3 --steps 8 --warmup 4 --no-cpu-baseline > $OUT/ncu_ff.log 2>&1; tail -2 $OUT/ncu_ff.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3_final.csv \
  python bench.py --workload c3 --steps 30 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
bash scripts/ncu_summary.sh $OUT/field_fused_c3_final.ncu-rep > $OUT/field_fused_c3_final.txt 2>&1
python scripts/launch_summary.py $OUT/launches_c3_final.csv "c3 final" > $OUT/launches_c3_final.txt 2>&1
head -30 $OUT/field_fused_c3_final.txt; head -8 $OUT/launches_c3_final.txt
