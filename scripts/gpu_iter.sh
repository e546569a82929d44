# Iteration loop: GPU tests, bench (TMA and LDG paths), ncu capture of the push kernel.
OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; tail -3 $OUT/pytest_gpu.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_tma.txt 2>&1
PB_PUSH_PATH=ldg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_ldg.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_push -s 4 -c 1 \
  -o $OUT/push_tma python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for f in bench_tma bench_ldg; do python -c "
import json,sys; d=json.loads(open('$OUT/$f.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4), 'frac', round(r['frac'],3))" || tail -5 $OUT/$f.txt; done
