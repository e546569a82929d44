# replay() graph length A/B (Engine.GRAPH_STEPS), interleaved, plus the replay parity tests at 10
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -c "
import sys, pytest
import paper_2404_10270_b200.engine as e
e.Engine.GRAPH_STEPS = 10
sys.exit(pytest.main(['-x', '-q', '-m', 'gpu', 'tests/test_fullsize_gpu.py', 'tests/test_engine_gpu.py', 'tests/test_field_cycle_gpu.py']))
" > $OUT/graph_tests.txt 2>&1; tail -2 $OUT/graph_tests.txt
run() { python -c "
import sys, runpy
import paper_2404_10270_b200.engine as e
e.Engine.GRAPH_STEPS = $2
sys.argv = ['bench.py', '--workload', '$1', '--steps', '400', '--warmup', '10', '--no-cpu-baseline']
runpy.run_path('bench.py', run_name='__main__')
" > $OUT/gab.txt 2>&1; python -c "
import json; d=json.loads(open('$OUT/gab.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$1 G=$2', round(d['value']/1e9,2), 'step', round(d['ms_per_step']*1e3,2), 'push', round(r['push_ms']*1e3,2), 'e2e', round(d['e2e']['value']/1e9,2))" || tail -3 $OUT/gab.txt; }
timeout 300 python bench.py --workload c3 --steps 100 --warmup 10 --no-cpu-baseline > /dev/null 2>&1
for r in 1 2; do for w in c3 c2; do for G in 2 10 24; do run $w $G; done; done; done
