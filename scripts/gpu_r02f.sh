OUT=gpurun_out
mkdir -p $OUT
timeout 900 python scripts/field_cycle_ab.py 65536 100000 > $OUT/field_cycle_ab.jsonl 2>&1; cat $OUT/field_cycle_ab.jsonl | tail -12
for v in nofence sleep; do
  PB_LIB_PATH=build/v_$v/libpicmc_b200.so timeout 900 python scripts/field_cycle_ab.py 65536 > $OUT/field_cycle_ab_$v.jsonl 2>&1; echo $v; cat $OUT/field_cycle_ab_$v.jsonl | tail -6
done
