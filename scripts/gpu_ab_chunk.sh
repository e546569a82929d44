# claim granularity A/B (PB_CHUNK_TARGET: chunks per warp; 0 = fixed 2048)
OUT=gpurun_out
for w in c3 c2 c4; do
  for t in 0 8 16 0 8 16; do
    PB_CHUNK_TARGET=$t timeout 900 python bench.py --workload $w --steps 400 --warmup 10 --no-cpu-baseline > $OUT/ck_${w}_$t.txt 2>&1
    echo "$w T=$t $(tail -1 $OUT/ck_${w}_$t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["ms_per_step"], d["roofline"]["push_ms"], d["roofline"]["frac"])')"
  done
done
