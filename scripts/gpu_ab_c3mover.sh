# config 3 mover variants: ring (int32 cell) vs split-solo (int32 / cell8) vs quad
OUT=gpurun_out
run() {
  env $2 timeout 900 python bench.py --workload c3 --steps 400 --warmup 10 --no-cpu-baseline > $OUT/c3m_$1.txt 2>&1
  echo "$1 [$2] $(tail -1 $OUT/c3m_$1.txt | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["value"]/1e9, d["ms_per_step"], d["roofline"]["push_ms"], d["roofline"]["kernel"])')"
}
for rep in 1 2; do
run ring PB_PDL=1
run solo_i32 PB_SPLIT_SOLO=1
run solo_c8 "PB_SPLIT_SOLO=1 PB_CELL8=2"
run quad_c8 "PB_RING=0 PB_CELL8=2"
run quad PB_RING=0
done
