# r02v: fp64 closed-form scan: parity, standalone + in-pipeline timelines, c3/c4 bench, graph_steps probe
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_field_cycle_gpu.py tests/test_harness_gpu.py -q -x -rf > $OUT/pytest_v.txt 2>&1; tail -3 $OUT/pytest_v.txt
python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so 65536
PB_LIB_PATH=build/v_fftrace/libpicmc_b200.so python scripts/c3_pipeline_trace.py
for w in c3 c4; do
timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_v_$w.txt 2>&1
python -c "
import json; d=json.loads(open('$OUT/bench_v_$w.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$w', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4))"
done
python scripts/graph_steps_probe.py c2 1000
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_fullsize_gpu.py tests/test_bfield_gpu.py -q -x -rf > $OUT/pytest_v2.txt 2>&1; tail -3 $OUT/pytest_v2.txt
