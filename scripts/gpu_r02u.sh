# r02u: tile_local / warp prefixes; standalone vs in-pipeline timeline with SM placement and clock
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_field_cycle_gpu.py tests/test_harness_gpu.py -q -x -rf > $OUT/pytest_u.txt 2>&1; tail -3 $OUT/pytest_u.txt
python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so 65536
PB_LIB_PATH=build/v_fftrace/libpicmc_b200.so python scripts/c3_pipeline_trace.py
timeout 600 python bench.py --workload c3 --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_u_c3.txt 2>&1
python -c "
import json; d=json.loads(open('$OUT/bench_u_c3.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('c3', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4))"
