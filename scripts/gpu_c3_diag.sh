OUT=gpurun_out
: > $OUT/c3diag.txt
for envs in "PB_CELL8=1" "PB_CELL8=0" "PB_CELL8=1"; do
  env $envs timeout 600 python bench.py --workload c3 --steps 400 --warmup 10 --no-cpu-baseline > $OUT/c3d.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/c3d.txt').read().strip().splitlines()[-1]); print('$envs', round(d['ms_per_step'],4), d['timing_windows_ms'])" >> $OUT/c3diag.txt || tail -3 $OUT/c3d.txt >> $OUT/c3diag.txt
done
cat $OUT/c3diag.txt
