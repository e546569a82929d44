# r02t: PDL trigger placement of k_field_fused (late = after the solve, default; early = at entry)
OUT=gpurun_out
mkdir -p $OUT
echo "late trigger:"; PB_LIB_PATH=build/v_fftrace/libpicmc_b200.so python scripts/c3_pipeline_trace.py
echo "early trigger:"; PB_LIB_PATH=build/v_fftrace_early/libpicmc_b200.so python scripts/c3_pipeline_trace.py
for v in base early base early; do
  lib=paper_2404_10270_b200/libpicmc_b200.so; [ $v = early ] && lib=build/v_early/libpicmc_b200.so
  PB_LIB_PATH=$lib timeout 600 python bench.py --workload c3 --steps 400 --warmup 20 --no-cpu-baseline > $OUT/bench_t_$v.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/bench_t_$v.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$v c3', round(d['value']/1e9,2),'Gpush/s', 'step ms', round(d['ms_per_step'],4), 'push ms', round(r['push_ms'],4))" || tail -3 $OUT/bench_t_$v.txt
done
python scripts/c2_gap_probe.py 1000
