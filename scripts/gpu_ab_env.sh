# bench under env settings x sort periods (no CPU baseline).
# lines of scripts/envs.txt: "<sort_every> <ENV=VAL ...>"
OUT=gpurun_out
: > $OUT/abenv.txt
i=0
while read -r se envs; do
  i=$((i+1))
  env $envs timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --sort-every $se > $OUT/b_env$i.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/b_env$i.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('sort=$se $envs', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2))" >> $OUT/abenv.txt 2>&1 || tail -3 $OUT/b_env$i.txt >> $OUT/abenv.txt
done < scripts/envs.txt
cat $OUT/abenv.txt
