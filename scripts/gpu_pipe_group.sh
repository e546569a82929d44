# A/B of run_pipelined block sizes (PB_PIPE_GROUP) on the e2e number
OUT=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "pipelined or pipe_graphs or absorbing or sort" > $OUT/pipe_tests.txt 2>&1
tail -3 $OUT/pipe_tests.txt
for w in c2 c3 c4; do
  for g in 1 4 8; do
    PB_PIPE_GROUP=$g timeout 900 python bench.py --workload $w --steps 400 --warmup 10 --no-cpu-baseline > $OUT/pg_${w}_$g.txt 2>&1
    echo "$w G=$g $(tail -1 $OUT/pg_${w}_$g.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["e2e"]["value"]/1e9, d["e2e"].get("graphs_captured_in_timed_region"), d["ms_per_step"])')"
  done
done
