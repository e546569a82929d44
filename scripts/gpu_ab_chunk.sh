# claim-chunk A/B (PB_CLAIM_CHUNK) + full GPU suite
OUT=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/ck_tests.txt 2>&1; tail -2 $OUT/ck_tests.txt
for w in c2 c4 c5 c3; do
  for t in 2048 1024 2048 1024; do
    PB_CLAIM_CHUNK=$t timeout 900 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline > $OUT/ck_${w}_$t.txt 2>&1
    echo "$w C=$t $(tail -1 $OUT/ck_${w}_$t.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["ms_per_step"], d["roofline"]["push_ms"], d["roofline"]["frac"])')"
  done
done
