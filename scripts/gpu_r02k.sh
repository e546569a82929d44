OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_field_cycle_gpu.py tests/test_fullsize_gpu.py tests/test_engine_gpu.py tests/test_harness_gpu.py tests/test_multirank_gpu.py -q -rf -x > $OUT/pytest_k.txt 2>&1; tail -4 $OUT/pytest_k.txt
timeout 600 python scripts/field_cycle_ab.py 65536 100000 > $OUT/field_cycle_ab_k.jsonl 2>&1; tail -8 $OUT/field_cycle_ab_k.jsonl
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_$w.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/bench_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac(push)', round(r['frac'],3), 'step frac', round(r['alg_bytes_per_launch']/d['ms_per_step']/1e6/r['peak'],3), r['kernel'], 'e2e', round(d['e2e']['value']/1e9,2))" || tail -5 $OUT/bench_$w.txt
done
