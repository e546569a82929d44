# config-3 (ring kernel) compile-time variants: EXTRA flags per line of
# scripts/ring_variants.txt (empty line = default build)
OUT=gpurun_out
mkdir -p /tmp/v
: > $OUT/ring_var.txt
i=0
while IFS= read -r flags; do
  i=$((i+1))
  make -s -C paper_2404_10270_b200/csrc OUT=/tmp/v/r$i.so BUILD=/tmp/v/rb$i EXTRA="$flags" > /tmp/v/rm$i 2>&1 || { tail -3 /tmp/v/rm$i >> $OUT/ring_var.txt; continue; }
  for rep in 1 2; do
    PB_LIB_PATH=/tmp/v/r$i.so timeout 300 python bench.py --workload c3 --steps 400 --warmup 10 --no-cpu-baseline > $OUT/rv.txt 2>&1
    python -c "
import json; d=json.loads(open('$OUT/rv.txt').read().strip().splitlines()[-1]); print('[$flags]', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['roofline']['push_ms'],4), d['roofline']['kernel'])" >> $OUT/ring_var.txt || tail -3 $OUT/rv.txt >> $OUT/ring_var.txt
  done
done < scripts/ring_variants.txt
cat $OUT/ring_var.txt
