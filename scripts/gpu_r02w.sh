# r02w: full -m gpu suite + field timelines + c3/c4 bench
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_w.txt 2>&1; tail -3 $OUT/pytest_w.txt
python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so 65536
python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so 100000 periodic
PB_LIB_PATH=build/v_fftrace/libpicmc_b200.so python scripts/c3_pipeline_trace.py
for w in c3 c4; do
timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_w_$w.txt 2>&1
python -c "
import json; d=json.loads(open('$OUT/bench_w_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4))"
done
