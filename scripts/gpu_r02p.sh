# r02p: k_field_fused without full fences: parity + c3/c4 bench + launch list
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_field_cycle_gpu.py -q -x -rf > $OUT/pytest_p.txt 2>&1; tail -3 $OUT/pytest_p.txt
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_p_$w.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/bench_p_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac(push)', round(r['frac'],3), 'step frac', round(r['alg_bytes_per_launch']/d['ms_per_step']/1e6/r['peak'],3), 'e2e', round(d['e2e']['value']/1e9,2))" || tail -5 $OUT/bench_p_$w.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3_p.csv \
  python bench.py --workload c3 --steps 30 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py $OUT/launches_c3_p.csv | head -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_field_fused -s 5 -c 1 \
  -o $OUT/field_fused_c3 python bench.py --workload c3 --steps 8 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
ls $OUT/field_fused_c3*
