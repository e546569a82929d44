OUT=gpurun_out
: > $OUT/ab_field.txt
for w in c3 c4; do for v in 1 0; do
  PB_FUSED_FIELD=$v timeout 600 python bench.py --workload $w --steps 400 --warmup 10 --no-cpu-baseline > $OUT/f_${w}_$v.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/f_${w}_$v.txt').read().strip().splitlines()[-1]); print('$w fused=$v', round(d['value']/1e9,2), round(d['ms_per_step'],4), d['gpu_launches'])" >> $OUT/ab_field.txt || tail -3 $OUT/f_${w}_$v.txt >> $OUT/ab_field.txt
done; done
cat $OUT/ab_field.txt
