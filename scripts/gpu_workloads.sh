# one bench line per BASELINE config (c2 default, c3, c4, c5) on one GPU
OUT=gpurun_out
for w in c2 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --steps 400 --warmup 10 --no-cpu-baseline > $OUT/wl_$w.txt 2>&1
  tail -1 $OUT/wl_$w.txt | cut -c1-300
done
