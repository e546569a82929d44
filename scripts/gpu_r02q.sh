# r02q: closed-form scan solve + single-launch field cycle: parity, timeline, c3/c4 bench
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_field_cycle_gpu.py tests/test_harness_gpu.py -q -x -rf > $OUT/pytest_r.txt 2>&1; tail -12 $OUT/pytest_r.txt
python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so 65536
python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so 100000 periodic
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_fullsize_gpu.py tests/test_bfield_gpu.py tests/test_multirank_gpu.py -q -x -rf > $OUT/pytest_r2.txt 2>&1; tail -5 $OUT/pytest_r2.txt
for w in c3 c4; do
  timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_r_$w.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/bench_r_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac(push)', round(r['frac'],3), 'step frac', round(r['alg_bytes_per_launch']/d['ms_per_step']/1e6/r['peak'],3), 'e2e', round(d['e2e']['value']/1e9,2))" || tail -5 $OUT/bench_r_$w.txt
done
