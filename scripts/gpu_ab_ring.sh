OUT=gpurun_out
: > $OUT/ab_ring.txt
for v in 1 0 1 0; do
  PB_RING=$v timeout 600 python bench.py --workload c3 --steps 400 --warmup 10 --no-cpu-baseline > $OUT/r_$v.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/r_$v.txt').read().strip().splitlines()[-1]); print('ring=$v', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['roofline']['push_ms'],4), d['timing_windows_ms']['max'])" >> $OUT/ab_ring.txt || tail -3 $OUT/r_$v.txt >> $OUT/ab_ring.txt
done
cat $OUT/ab_ring.txt
