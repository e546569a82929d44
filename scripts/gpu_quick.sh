OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; tail -3 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py --steps 40 --warmup 6 --no-cpu-baseline > $OUT/bench.txt 2>&1
python -c "
import json; d=json.loads(open('$OUT/bench.txt').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), 'SOL ms', round(d['sol_probe']['ms'],4))" || tail -5 $OUT/bench.txt
