# config-3 run_simulation leg variance: four bench runs, wall vs device seconds of the leg
OUT=gpurun_out; mkdir -p $OUT
for r in 1 2 3 4 5 6; do
  timeout 600 python bench.py --workload c3 --steps 400 --warmup 10 --no-cpu-baseline > $OUT/rsv_$r.txt 2>&1
  tail -1 $OUT/rsv_$r.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e_run_simulation']
print('run $r value', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2), 'rs', round(e['value']/1e9,2), 'wall_s', round(e['wall_s'],4), 'device_s', round(e['device_s'],4))"
done
