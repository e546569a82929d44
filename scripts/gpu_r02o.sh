# r02o: single-launch field cycle (k_field_fused): parity + c3/c4 bench
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_field_cycle_gpu.py -q -x -rf > $OUT/pytest_o.txt 2>&1; tail -15 $OUT/pytest_o.txt
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_harness_gpu.py tests/test_fullsize_gpu.py tests/test_bfield_gpu.py -q -x -rf > $OUT/pytest_o2.txt 2>&1; tail -5 $OUT/pytest_o2.txt
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_o_$w.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/bench_o_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac(push)', round(r['frac'],3), 'step frac', round(r['alg_bytes_per_launch']/d['ms_per_step']/1e6/r['peak'],3), 'e2e', round(d['e2e']['value']/1e9,2))" || tail -5 $OUT/bench_o_$w.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3_o.csv \
  python bench.py --workload c3 --steps 30 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py $OUT/launches_c3_o.csv | head -14
