# programmatic dependent launch A/B (PB_PDL)
OUT=gpurun_out
for w in c3 c4 c2; do
  for p in 0 1 0 1; do
    PB_PDL=$p timeout 900 python bench.py --workload $w --steps 400 --warmup 10 --no-cpu-baseline > $OUT/pdl_${w}_$p.txt 2>&1
    echo "$w PDL=$p $(tail -1 $OUT/pdl_${w}_$p.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["e2e"]["value"]/1e9, d["ms_per_step"], d["roofline"]["push_ms"])')"
  done
done
