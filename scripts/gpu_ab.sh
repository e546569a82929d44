# Interleaved A/B of library builds: bash scripts/gpu_ab.sh "c2 c3" base:paper_2404_10270_b200/libpicmc_b200.so v1:build/v_x/libpicmc_b200.so ...
# One throwaway warm-up bench, then two rounds over the variants (a fresh box's first runs are slow).
OUT=gpurun_out; mkdir -p $OUT
WL="$1"; shift
summ() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
print(sys.argv[2], sys.argv[3], round(d['value']/1e9,2),'Gpush/s step', round(d['ms_per_step']*1e3,2),'us push', round(r['push_ms']*1e3,2), 'us frac', round(r['frac'],3))" "$@" || tail -3 "$1"; }
timeout 300 python bench.py --workload c2 --steps 100 --warmup 10 --no-cpu-baseline > /dev/null 2>&1
for round in 1 2; do
  for w in $WL; do
    for v in "$@"; do
      name=${v%%:*}; lib=${v#*:}
      PB_LIB_PATH=$lib timeout 600 python bench.py --workload $w --steps 400 --warmup 20 --no-cpu-baseline > $OUT/ab_${name}_${w}_$round.txt 2>&1
      summ $OUT/ab_${name}_${w}_$round.txt $w $name
    done
  done
done
