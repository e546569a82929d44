# bench value vs sort period (no CPU baseline)
OUT=gpurun_out
: > $OUT/sortsweep.txt
for se in 0 25 50 100 200; do
  timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --sort-every $se > $OUT/b_$se.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/b_$se.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('sort_every=$se', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac', round(r['frac'],3))" >> $OUT/sortsweep.txt 2>&1 || tail -3 $OUT/b_$se.txt >> $OUT/sortsweep.txt
done
cat $OUT/sortsweep.txt
