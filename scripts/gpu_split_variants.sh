OUT=gpurun_out
mkdir -p /tmp/v
: > $OUT/split_var.txt
i=0
while IFS= read -r flags; do
  i=$((i+1))
  make -s -C paper_2404_10270_b200/csrc OUT=/tmp/v/s$i.so BUILD=/tmp/v/sb$i EXTRA="$flags" > /tmp/v/sm$i 2>&1 || { tail -3 /tmp/v/sm$i >> $OUT/split_var.txt; continue; }
  PB_SPLIT=1 PB_LIB_PATH=/tmp/v/s$i.so timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > $OUT/sv.txt 2>&1
  python -c "
import json; d=json.loads(open('$OUT/sv.txt').read().strip().splitlines()[-1]); print('$flags', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['roofline']['push_ms'],4))" >> $OUT/split_var.txt || tail -3 $OUT/sv.txt >> $OUT/split_var.txt
done < scripts/split_variants.txt
PB_SPLIT=0 timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > $OUT/sv.txt 2>&1
python -c "
import json; d=json.loads(open('$OUT/sv.txt').read().strip().splitlines()[-1]); print('nosplit', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['roofline']['push_ms'],4))" >> $OUT/split_var.txt
cat $OUT/split_var.txt
