# compile-time variants on one workload: bash scripts/gpu_variants.sh <c2|c3|c4|c5> <variants file>
# (one EXTRA flag set per line, empty line = default build).  One throwaway
# warm-up run first (a fresh box's first runs are slower), then two rounds
# over all variants, interleaved.
OUT=gpurun_out
W=$1; V=$2
mkdir -p /tmp/v
: > $OUT/var_$W.txt
mapfile -t FLAGS < $V
for i in "${!FLAGS[@]}"; do
  make -s -C paper_2404_10270_b200/csrc OUT=/tmp/v/x$i.so BUILD=/tmp/v/xb$i EXTRA="${FLAGS[$i]}" > /tmp/v/xm$i 2>&1 || tail -3 /tmp/v/xm$i >> $OUT/var_$W.txt
done
timeout 300 python bench.py --workload $W --steps 400 --warmup 10 --no-cpu-baseline > /dev/null 2>&1
for rep in 1 2; do
  for i in "${!FLAGS[@]}"; do
    PB_LIB_PATH=/tmp/v/x$i.so timeout 300 python bench.py --workload $W --steps 400 --warmup 10 --no-cpu-baseline > $OUT/xv.txt 2>&1
    python -c "
import json; d=json.loads(open('$OUT/xv.txt').read().strip().splitlines()[-1]); print('[${FLAGS[$i]}]', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['roofline']['push_ms'],4), d['roofline']['kernel'])" >> $OUT/var_$W.txt || tail -3 $OUT/xv.txt >> $OUT/var_$W.txt
  done
done
cat $OUT/var_$W.txt
