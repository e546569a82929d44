OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_field_cycle_gpu.py tests/test_fullsize_gpu.py tests/test_engine_gpu.py tests/test_harness_gpu.py -q -rf -x > $OUT/pytest_e.txt 2>&1; tail -8 $OUT/pytest_e.txt
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_$w.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/bench_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac(push)', round(r['frac'],3), 'step frac', round(r['alg_bytes_per_launch']/d['ms_per_step']/1e6/r['peak'],3), r['kernel'], 'e2e', round(d['e2e']['value']/1e9,2))" || tail -5 $OUT/bench_$w.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv python bench.py --workload c3 --steps 6 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/launches_c3.csv')))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(list)
for r in rows[hdr+1:]:
    if len(r) > vi: agg[r[ki][:60]].append(float(r[vi].replace(',', '')))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:14]:
    print(f"{len(v):5d} {sum(v)/len(v)/1e3:9.2f} us  {k}")
PY
