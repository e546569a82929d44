# r02: gathered-B Boris tests + c4 / c4b bench lines
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_bfield_gpu.py tests/test_canonical_gpu.py tests/test_engine_gpu.py tests/test_mover_property_gpu.py -q -rf -x > $OUT/pytest_b.txt 2>&1; tail -15 $OUT/pytest_b.txt
for w in c4 c4b; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline > $OUT/bench_$w.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/bench_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac', round(r['frac'],3), r['kernel'], 'e2e', round(d['e2e']['value']/1e9,2), 'SOL ms', round(d['sol_probe']['ms'],4))" || tail -5 $OUT/bench_$w.txt
done
