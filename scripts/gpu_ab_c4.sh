OUT=gpurun_out
: > $OUT/ab_c4.txt
for v in 1 0 1 0; do
  PB_FIELD_SPLIT=$v timeout 600 python bench.py --workload c4 --steps 400 --warmup 10 --no-cpu-baseline > $OUT/c4_$v.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/c4_$v.txt').read().strip().splitlines()[-1]); print('split=$v', round(d['value']/1e9,2), round(d['ms_per_step'],4))" >> $OUT/ab_c4.txt
done
cat $OUT/ab_c4.txt
