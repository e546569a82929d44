# run_simulation status-check interval A/B (PB_CHECK_EVERY 128 vs 512), c3 and c2, interleaved
OUT=gpurun_out; mkdir -p $OUT
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], 'value', round(d['value']/1e9,2), 'e2e', round(d['e2e']['value']/1e9,2), 'run_simulation', round(d['e2e_run_simulation']['value']/1e9,2), d['e2e_run_simulation']['steps'])" "$@" || tail -3 "$1"; }
timeout 300 python bench.py --workload c3 --steps 100 --warmup 10 --no-cpu-baseline > /dev/null 2>&1
for r in 1 2; do
  for w in c3 c2; do
    for c in 128 512; do
      PB_CHECK_EVERY=$c timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/ck_${w}_${c}_$r.txt 2>&1
      summ $OUT/ck_${w}_${c}_$r.txt "$w check=$c r$r"
    done
  done
done
PB_CHECK_EVERY=512 timeout 600 python bench.py --workload c3 --steps 2000 --warmup 20 --no-cpu-baseline > $OUT/ck_c3_512_long.txt 2>&1; summ $OUT/ck_c3_512_long.txt "c3 check=512 2000 steps"
PB_CHECK_EVERY=128 timeout 600 python bench.py --workload c3 --steps 2000 --warmup 20 --no-cpu-baseline > $OUT/ck_c3_128_long.txt 2>&1; summ $OUT/ck_c3_128_long.txt "c3 check=128 2000 steps"
